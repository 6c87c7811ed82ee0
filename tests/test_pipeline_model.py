"""The paper's pipeline cost model (include/helmsweep/pipeline.hpp, src/pipeline.cpp:20-111) in
the product library against the reference's own average_time_per_rhs / simulate_pipeline
(oracle/_ref). Host-only."""
import ctypes

import numpy as np
import pytest

import paper_2003_02585_b200 as hs
from oracle import ref as R

SCENARIOS = [(2, [4, 4], 1, 1, 1.0), (2, [8, 8], 16, 1, 0.37), (2, [3, 2], 5, 2, 2.5), (3, [2, 2, 2], 4, 1, 1.0),
             (2, [8, 8], 15, 1, 1.0), (3, [4, 4, 4], 8, 1, 0.125), (2, [5, 1], 7, 3, 1.0)]


@pytest.mark.parametrize("dim,counts,n_rhs,n_iter,t0", SCENARIOS)
def test_pipeline_model_matches_reference(dim, counts, n_rhs, n_iter, t0):
    if not R.available():
        pytest.skip("oracle/_ref not built")
    L = R.lib()
    d = [ctypes.c_double() for _ in range(4)]
    comp = np.zeros(n_rhs)
    c3 = (ctypes.c_int * 3)(*(counts + [1, 1])[:3])
    rc = L.hsref_pipeline(dim, c3, n_rhs, n_iter, ctypes.c_double(t0), *[ctypes.byref(x) for x in d],
                          comp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert rc == 0
    cost = hs.average_time_per_rhs(dim, counts, n_rhs, n_iter, t0)
    sim = hs.simulate_pipeline(dim, counts, n_rhs, n_iter, t0)
    assert cost.average_per_rhs == d[0].value and cost.idle_fraction == d[1].value
    assert sim.makespan == d[2].value and sim.average_per_rhs == d[3].value
    np.testing.assert_array_equal(sim.completion_times, comp)


def test_pipeline_model_rejects_bad_scenarios():
    with pytest.raises(hs.ConfigError):
        hs.average_time_per_rhs(4, [2, 2], 1, 1, 1.0)
    with pytest.raises(hs.ConfigError):
        hs.simulate_pipeline(2, [2, 2], 0, 1, 1.0)
