"""CPU: the numpy oracle (oracle/hs_oracle.py) pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py) and against the reference's own known-answer
tests (tests/test_direct.cpp)."""
import ast
import math

import numpy as np
import pytest

from oracle import hs_oracle as O

COUNTERS = ["traces_generated", "traces_routed", "traces_discarded", "local_solves", "skipped_zero_solves"]

# SURVEY.md Appendix B (reference route_trace output), columns (-x, +x, -y, +y[, -z, +z])
APPENDIX_B = {
    (2, 1): [[2, 1, 3, 1], [2, 0, 4, 2], [4, 3, 3, 0], [4, 0, 4, 0]],
    (2, 2): [[2, 1, 3, 1], [2, 5, 4, 2], [4, 3, 3, 5], [4, 7, 4, 6], [6, 5, 7, 5], [6, 0, 8, 6], [8, 7, 7, 0],
             [8, 0, 8, 0]],
    (3, 1): [[2, 1, 3, 1, 5, 1], [2, 0, 4, 2, 6, 2], [4, 3, 3, 0, 7, 3], [4, 0, 4, 0, 8, 4], [6, 5, 7, 5, 5, 0],
             [6, 0, 8, 6, 6, 0], [8, 7, 7, 0, 7, 0], [8, 0, 8, 0, 8, 0]],
}


def oracle_route_table(dim, rounds):
    plan = O.sweep_plan(dim, rounds)
    return np.array([[O.route_trace(plan, dim, l, d // 2, 1 if d & 1 else -1) for d in range(2 * dim)]
                     for l in range(1, len(plan) + 1)])


@pytest.mark.parametrize("dim,rounds", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_routing_matches_reference(golden, dim, rounds):
    tab = oracle_route_table(dim, rounds)
    assert np.array_equal(tab, golden("routing")[f"route_{dim}d_r{rounds}"])
    if (dim, rounds) in APPENDIX_B:
        assert tab.tolist() == APPENDIX_B[(dim, rounds)]


def test_step_groups_cover_partition():
    part = O.Partition(O.Box(2), [64, 63], [4, 3])
    for d in O.ORDER2:
        seen = []
        for s in range(1, O.sweep_step_count(part.counts, 2) + 1):
            g = O.step_group(part, d, s)
            ids = [part.flatten(x) for x in g]
            assert ids == sorted(ids)
            seen += ids
        assert sorted(seen) == list(range(12))
    with pytest.raises(O.ConfigError):
        O.step_group(part, O.ORDER2[0], 0)


def _csr(z):
    return O.Csr(len(z["row_ptr"]) - 1, z["row_ptr"], z["col"], z["val"])


@pytest.mark.parametrize("name", ["direct_2d", "direct_3d", "direct_2d_16"])
def test_direct_solve_golden(golden, name):
    z = golden(name)
    dim = int(z["dim"])
    op = _csr(z)
    f = O.factorize(op, dim, O.GridRange(dim, list(z["lo"]), list(z["hi"])))
    assert f.factor_nnz == int(z["factor_nnz"])
    assert f.factor_nnz > op.n
    x = f.solve(z["b"])
    assert np.linalg.norm(x - z["x"]) / np.linalg.norm(z["x"]) <= 1e-12
    r = np.linalg.norm(op.apply(x) - z["b"]) / np.linalg.norm(z["b"])
    assert r <= 1e-10  # tests/test_direct.cpp:95-104
    assert np.array_equal(x, f.solve(z["b"]))  # bitwise repeatable (test_direct.cpp:123-134)


def _diag_op(d):
    n = len(d)
    return O.Csr(n, np.arange(n + 1), np.arange(n), np.array(d, dtype=np.complex128)), O.GridRange(2, [0, 0, 0], [n - 1, 0, 0])


def test_known_answers():
    op, rng = _diag_op([2.0])  # tests/test_direct.cpp:77-86
    assert O.factorize(op, 2, rng).solve(np.array([3 + 1j]))[0] == 1.5 + 0.5j
    op, rng = _diag_op([1.0] * 5)
    b = np.arange(5) + 1j
    assert np.array_equal(O.factorize(op, 2, rng).solve(b), b)
    op, rng = _diag_op([1.0, 0.0, 1.0])  # test_direct.cpp:136-144
    with pytest.raises(O.SingularMatrixError) as e:
        O.factorize(op, 2, rng)
    assert e.value.pivot_index == 1


def _setup_from(z):
    dim = int(z["dim"])
    med = ast.literal_eval(str(z["medium"]))
    kind = med["media.kind"]
    if kind == "constant":
        m = O.Medium("constant", kappa=med["media.kappa"])
    else:
        m = O.Medium("two_layered", kappa_down=med["media.kappa_down"], kappa_up=med["media.kappa_up"],
                     axis=med["media.axis"], eta=med["media.eta_L"], eps=med["media.epsilon"])
    n = int(z["n"])
    parts = list(z["parts"])
    return O.ProblemSetup(O.Box(dim), [n] * dim + [1] * (3 - dim), parts + [1] * (3 - dim), m,
                          O.PmlSpec(width=int(z["pad"])))


@pytest.mark.parametrize("name", ["ddm_2d_2x2", "ddm_2d_3x2_r2", "ddm_2d_layered", "ddm_3d_2x2x2"])
def test_ddm_golden(golden, name):
    z = golden(name)
    s = O.DdmSolver(_setup_from(z))
    assert [st.fact.factor_nnz for st in s.states] == list(z["factor_nnz"])
    assert [st.fact.peak_bytes for st in s.states] == list(z["peak_bytes"])
    for r in range(z["b"].shape[0]):
        u, rep = s.ddm_solve(z["b"][r].copy(), int(z["rounds"]), True)
        assert np.linalg.norm(u - z["u"][r]) / np.linalg.norm(z["u"][r]) <= 1e-10
        assert [getattr(rep, k) for k in COUNTERS] == list(z["counters"][r])
        np.testing.assert_allclose(rep.sweep_contrib_norm, z["contrib_norm"][r], rtol=1e-9)
        np.testing.assert_allclose(rep.round_residuals, z["round_residuals"][r], rtol=1e-7)


def test_ddm_linearity_and_zero():
    z = None
    setup = O.ProblemSetup(O.Box(2), [32, 32, 1], [2, 2, 1], O.Medium("constant", kappa=6 * math.pi), O.PmlSpec(width=6))
    s = O.DdmSolver(setup)
    f = O.gaussian_source(s.ggrid, O.Box(2), [[0.3, 0.3], [0.7, 0.4]], 2.0 / 32)
    b = s.scale_source(f)
    u0, _ = s.ddm_solve(b[:, 0].copy(), 1)
    u1, _ = s.ddm_solve(b[:, 1].copy(), 1)
    u01, _ = s.ddm_solve((2.0 * b[:, 0] - 1j * b[:, 1]).copy(), 1)
    assert np.linalg.norm(u01 - (2.0 * u0 - 1j * u1)) / np.linalg.norm(u01) <= 1e-12  # SPEC linearity
    uz, rep = s.ddm_solve(np.zeros_like(b[:, 0]), 1)
    assert not np.any(uz) and rep.local_solves == 0 and rep.skipped_zero_solves == 4 * 4
    del z


def test_gmres_golden(golden):
    z = golden("gmres_2d")
    setup = O.ProblemSetup(O.Box(2), [int(z["n"])] * 2 + [1], list(z["parts"]) + [1],
                           O.Medium("constant", kappa=ast.literal_eval(str(z["medium"]))["media.kappa"]),
                           O.PmlSpec(width=int(z["pad"])))
    s = O.DdmSolver(setup)
    g = O.gmres(lambda v: s.global_op().apply(v), lambda v: s.ddm_solve(v, 1)[0], z["b"].copy(),
                float(z["tol"]), int(z["maxit"]))
    assert abs(g.iterations - int(z["iterations"])) <= 1
    assert g.true_residual <= 10 * float(z["true_residual"]) + 1e-12
    assert np.linalg.norm(g.x - z["x"]) / np.linalg.norm(z["x"]) <= 1e-7
