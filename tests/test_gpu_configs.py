"""GPU parity at the BASELINE configurations themselves (BASELINE.json configs[0..4]), through the
C-ABI against the reference: oracle/_ref (the unmodified reference compiled in place, run on the
GPU box's host cores) where it fits the host, and the reference-generated golden fixture for C5's
subdomain size (tests/golden/make_c5_reduced.py) where it does not.

North-star bar: u within 1e-9 relative L2 (complex128), SolveReport counters bit-exact, per-round
residuals equal to roundoff, per-subdomain factor_nnz exact (src/direct.cpp:333-348).
"""
import hashlib
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

COUNTERS = ["traces_generated", "traces_routed", "traces_discarded", "local_solves", "skipped_zero_solves"]
TOL = 1e-9


@pytest.fixture(scope="module")
def hs():
    import paper_2003_02585_b200 as m
    if m.device_count() == 0:
        pytest.fail("gpu test run without a CUDA device")
    return m


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as r
    if not r.available():
        pytest.fail("oracle/_ref (the reference compiled in place) is missing: the config pins need it")
    return r


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _check_against_reference(hs, ref, cfg_name, nrhs_check=1):
    import bench
    bench.select(cfg_name)
    C = bench.CFG
    s = hs.DdmSolver(hs.ProblemSetup(2, [C["n"]] * 2, list(C["parts"]), bench.medium(hs), pml_width=C["pad"]))
    r = ref.RefSolver(bench.ref_config(), os.cpu_count())
    f = bench.make_sources(C["seed"], s.lo, s.hi, [1.0 / C["n"]] * 2, [0.0, 0.0])[:nrhs_check]
    b = s.scale_source(f)
    for i in range(nrhs_check):
        assert np.array_equal(b[i], r.scale_source(f[i]))  # DdmSolver::scale_source, bit for bit
    reps = []
    U = s.ddm_solve(b, C["rounds"], reps, True)
    for i in range(nrhs_check):
        u0, rep0 = r.ddm_solve(b[i], C["rounds"], True)
        assert rel(U[i], u0) <= TOL
        assert [getattr(reps[i], k) for k in COUNTERS] == [rep0[k] for k in COUNTERS]
        assert np.allclose(reps[i].round_residuals, rep0["round_residuals"], rtol=1e-9, atol=0)
        assert np.allclose(reps[i].sweep_contrib_norm, rep0["sweep_contrib_norm"], rtol=1e-8, atol=1e-300)
    for sub in (0, 1, s.nsub // 2, s.nsub - 1):
        assert s.sub_stats(sub).factor_nnz == r.sub_info(sub)["factor_nnz"]
    return s, b, U


def test_c2_full_scale_against_reference(hs, ref):
    """BASELINE configs[1] (C2) at full scale: 1024^2 + 32 PML, 8x8 subdomains, 1 round."""
    _check_against_reference(hs, ref, "c2")


def test_c3_full_scale_against_reference(hs, ref):
    """BASELINE configs[2] (C3, the bench headline) at full scale: 2048^2 two-layered medium,
    16x16 subdomains of 193^2, 2 rounds = 8 sweeps; RHS 0 of the bench's seeded batch."""
    s, b, U = _check_against_reference(hs, ref, "c3")
    # the same RHS inside the full 64-RHS batch gives the same u (to roundoff: the split-K shape of
    # the critical path depends on the batch width, and the order of the partial sums with it)
    import bench
    f = bench.make_sources(bench.CFG["seed"], s.lo, s.hi, [1.0 / bench.CFG["n"]] * 2, [0.0, 0.0])
    B = s.scale_source(f)
    assert np.array_equal(B[0], b[0])
    U64 = s.ddm_solve(B, bench.CFG["rounds"], None, True)
    assert rel(U64[0], U[0]) <= 1e-12


def test_c5_subdomain_size_against_reference_golden(hs, golden):
    """BASELINE configs[4] (C5) at its own subdomain size: 57^3 local grids (fronts up to
    m = 4845, k = 3249, the big-front cluster/DMMA factorization path), 2x2x2 subdomains on
    interior [0, 0.5]^3 with h = 1/128, kappa = 2 pi 12, 8 sweeps, against the reference's u
    (tests/golden/make_c5_reduced.py)."""
    from paper_2003_02585_b200 import sources
    z = golden("ddm_3d_c5_reduced")
    med = hs.Medium("constant", kappa=2 * math.pi * 12)
    s = hs.DdmSolver(hs.ProblemSetup(3, [64, 64, 64], [2, 2, 2], med, pml_width=12,
                                     interior_lo=(0.0, 0.0, 0.0), interior_hi=(0.5, 0.5, 0.5)))
    assert list(s.lo) == list(z["lo"]) and list(s.hi) == list(z["hi"])
    assert [s.sub_stats(i).factor_nnz for i in range(s.nsub)] == list(z["factor_nnz"])
    assert [s.sub_stats(i).peak_bytes for i in range(s.nsub)] == list(z["peak_bytes"])
    h = 0.5 / 64
    f = sources.gaussian_sources(3, s.lo, s.hi, [h] * 3, [0.0] * 3, z["centers"].tolist(), float(z["sigma"]),
                                 interior_lo=(0.0,) * 3, interior_hi=(0.5,) * 3)
    b = s.scale_source(f)
    assert hashlib.sha256(np.ascontiguousarray(b[0]).tobytes()).hexdigest() == str(z["b_sha256"])
    reps = []
    U = s.ddm_solve(b, 1, reps, True)
    assert rel(U[0], z["u"]) <= TOL
    assert [getattr(reps[0], k) for k in COUNTERS] == list(z["counters"])
    assert np.allclose(reps[0].round_residuals, z["round_residuals"], rtol=1e-9, atol=0)
    assert np.allclose(reps[0].sweep_contrib_norm, z["contrib_norm"], rtol=1e-8, atol=1e-300)
