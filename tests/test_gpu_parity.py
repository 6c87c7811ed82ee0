"""GPU parity: the B200 path (through the C-ABI, libhelmsweep_b200.so) against the reference's
golden vectors (tests/golden, produced by the reference itself) and the numpy oracle.

Tolerances (BASELINE.json north_star): solutions <= 1e-9 relative L2 in complex128; sweep /
trace counters bit-exact; GMRES iteration counts within +-1. The reference's own pins
(tests/test_direct.cpp) keep their tolerances (1e-10 residual, exact known answers)."""
import ast
import math

import numpy as np
import pytest

from oracle import hs_oracle as O

pytestmark = pytest.mark.gpu

COUNTERS = ["traces_generated", "traces_routed", "traces_discarded", "local_solves", "skipped_zero_solves"]
TOL = 1e-9


@pytest.fixture(scope="module")
def hs():
    import paper_2003_02585_b200 as m
    if m.device_count() == 0:
        pytest.fail("gpu test run without a CUDA device")
    return m


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def sparse_op(hs, z):
    dim = int(z["dim"])
    return hs.SparseOperator(dim, list(z["lo"]), list(z["hi"]), z["row_ptr"], z["col"], z["val"])


@pytest.mark.parametrize("name", ["direct_2d", "direct_3d", "direct_2d_16"])
def test_factor_solve_matches_reference(hs, golden, name):
    z = golden(name)
    op = sparse_op(hs, z)
    f = hs.factorize(op)
    assert f.stats().factor_nnz == int(z["factor_nnz"])
    x = f.solve(z["b"])
    assert rel(x, z["x"]) <= 1e-12
    A = O.Csr(op.n, z["row_ptr"], z["col"], z["val"])
    assert rel(A.apply(x), z["b"]) <= 1e-10            # tests/test_direct.cpp:95-104
    assert np.array_equal(x, f.solve(z["b"]))          # bitwise repeatable (:123-134)
    g = hs.factorize(op)
    assert np.array_equal(x, g.solve(z["b"]))          # re-factorization identical
    assert not np.any(f.solve(np.zeros(op.n, complex)))  # zero rhs -> exact zero (:88-93)


def test_forward_multiply_oracle(hs, golden):
    z = golden("direct_2d")  # tests/test_direct.cpp:106-121 (shell entries zeroed)
    op = sparse_op(hs, z)
    A = O.Csr(op.n, z["row_ptr"], z["col"], z["val"])
    rng = O.GridRange(2, list(z["lo"]), list(z["hi"]))
    P = rng.coords()
    shell = np.zeros(op.n, bool)
    for a in range(2):
        shell |= (P[a] == rng.lo[a]) | (P[a] == rng.hi[a])
    g = np.random.default_rng(21)
    xt = g.uniform(-1, 1, op.n) + 1j * g.uniform(-1, 1, op.n)
    xt[shell] = 0
    x = hs.factorize(op).solve(A.apply(xt))
    assert rel(x, xt) <= 1e-10


def test_known_answers(hs):
    one = hs.SparseOperator(2, [0, 0, 0], [0, 0, 0], np.array([0, 1]), np.array([0]), np.array([2.0 + 0j]))
    assert hs.factorize(one).solve(np.array([3 + 1j]))[0] == 1.5 + 0.5j
    n = 5
    ident = hs.SparseOperator(2, [0, 0, 0], [n - 1, 0, 0], np.arange(n + 1), np.arange(n), np.ones(n, complex))
    b = np.arange(n) + 0.5j
    assert np.array_equal(hs.factorize(ident).solve(b), b)
    bad = hs.SparseOperator(2, [0, 0, 0], [2, 0, 0], np.arange(4), np.arange(3), np.array([1.0, 0.0, 1.0], complex))
    with pytest.raises(hs.SingularMatrixError) as e:
        hs.factorize(bad)
    assert e.value.pivot_index == 1                     # tests/test_direct.cpp:136-144
    with pytest.raises(hs.ConfigError):
        hs.factorize(one).solve(np.zeros(3, complex))


def test_batched_solve_equals_single(hs, golden):
    z = golden("direct_3d")
    f = hs.factorize(sparse_op(hs, z))
    g = np.random.default_rng(3)
    B = g.standard_normal((7, f.stats().n)) + 1j * g.standard_normal((7, f.stats().n))
    B[4] = 0
    X = f.solve(B)
    for i in range(7):
        if i == 4:
            assert not np.any(X[i])
        else:
            assert rel(X[i], f.solve(B[i])) <= 1e-14


def _setup(hs, z):
    dim = int(z["dim"])
    med = ast.literal_eval(str(z["medium"]))
    if med["media.kind"] == "constant":
        m = hs.Medium("constant", kappa=med["media.kappa"])
    else:
        m = hs.Medium("two_layered", kappa_down=med["media.kappa_down"], kappa_up=med["media.kappa_up"],
                      axis=med["media.axis"], eta=med["media.eta_L"], eps=med["media.epsilon"])
    return hs.ProblemSetup(dim, [int(z["n"])] * dim, list(z["parts"]), m, pml_width=int(z["pad"]))


@pytest.mark.parametrize("name", ["ddm_2d_2x2", "ddm_2d_3x2_r2", "ddm_2d_layered", "ddm_3d_2x2x2"])
@pytest.mark.parametrize("batched", [False, True])
def test_ddm_matches_reference(hs, golden, name, batched):
    z = golden(name)
    s = hs.DdmSolver(_setup(hs, z))
    assert [s.sub_stats(i).factor_nnz for i in range(s.nsub)] == list(z["factor_nnz"])
    assert [s.sub_stats(i).peak_bytes for i in range(s.nsub)] == list(z["peak_bytes"])
    rounds = int(z["rounds"])
    R = z["b"].shape[0]
    if batched:
        reps = []
        U = s.ddm_solve(z["b"], rounds, reps, True)
    else:
        U, reps = [], []
        for r in range(R):
            U.append(s.ddm_solve(z["b"][r], rounds, reps, True))
    for r in range(R):
        assert rel(U[r], z["u"][r]) <= TOL
        assert [getattr(reps[r], k) for k in COUNTERS] == list(z["counters"][r])
        np.testing.assert_allclose(reps[r].sweep_contrib_norm, z["contrib_norm"][r], rtol=1e-8)
        np.testing.assert_allclose(reps[r].round_residuals, z["round_residuals"][r], rtol=1e-6)


def test_ddm_deterministic_and_linear(hs, golden):
    z = golden("ddm_2d_2x2")
    s = hs.DdmSolver(_setup(hs, z))
    b0, b1 = z["b"][0], z["b"][1]
    u = s.ddm_solve(np.stack([b0, b1, 2 * b0 - 1j * b1]), 1)
    assert np.array_equal(u[:2], s.ddm_solve(np.stack([b0, b1]), 1))  # bitwise across calls
    assert rel(u[2], 2 * u[0] - 1j * u[1]) <= 1e-12
    uz = []
    rz = s.ddm_solve(np.zeros_like(b0), 1, uz)
    assert not np.any(rz) and uz[0].local_solves == 0 and uz[0].skipped_zero_solves == 16


def test_c1_config_against_oracle(hs):
    """BASELINE config 1 (256^2, 4x4, PML 20, omega = 2 pi 16, centre source) and one seeded
    off-centre source, batched, against the numpy restatement."""
    n, pad, kap = 256, 20, 2 * math.pi * 16
    so = O.DdmSolver(O.ProblemSetup(O.Box(2), [n, n, 1], [4, 4, 1], O.Medium("constant", kappa=kap),
                                    O.PmlSpec(width=pad)))
    f = O.gaussian_source(so.ggrid, O.Box(2), [[0.5, 0.5], [0.3125, 0.6]], 2.0 / n)
    b = so.scale_source(f).T.copy()
    s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [4, 4], hs.Medium("constant", kappa=kap), pml_width=pad))
    reps = []
    U = s.ddm_solve(b, 1, reps, True)
    for r in range(2):
        uo, ro = so.ddm_solve(b[r].copy(), 1, True)
        assert rel(U[r], uo) <= TOL
        assert [getattr(reps[r], k) for k in COUNTERS] == [getattr(ro, k) for k in COUNTERS]
    assert [reps[0].local_solves, reps[0].skipped_zero_solves] == [48, 16]  # SURVEY §6.2 (C1 centre)


def test_gmres_matches_reference(hs, golden):
    z = golden("gmres_2d")
    med = ast.literal_eval(str(z["medium"]))
    s = hs.DdmSolver(hs.ProblemSetup(2, [int(z["n"])] * 2, list(z["parts"]), hs.Medium("constant", kappa=med["media.kappa"]),
                                     pml_width=int(z["pad"])))
    g = s.gmres(z["b"], float(z["tol"]), int(z["maxit"]), 1)
    assert abs(g.iterations - int(z["iterations"])) <= 1
    assert g.converged
    assert rel(g.x, z["x"]) <= 1e-7
    assert g.true_residual <= 1e-7


def test_general_gmres_seam(hs, golden):
    """gmres(op, pc, b, cfg) for caller-supplied LinearOperators (include/helmsweep/krylov.hpp:30-36)
    through hs_gmres_general: a dense operator with and without a right preconditioner against the
    oracle's restatement of src/krylov.cpp (same iteration counts and histories) and numpy's solve;
    then the reference's own wiring -- global operator and DDM application as host callbacks --
    against hs_gmres and the reference's golden GMRES run."""
    from oracle import hs_oracle as O
    g = np.random.default_rng(5)
    n = 300
    A = np.eye(n) * 4.0 + (g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))) / np.sqrt(n)
    Dinv = 1.0 / np.diag(A)
    B = g.standard_normal((3, n)) + 1j * g.standard_normal((3, n))
    B[2] = 0.0  # a zero right-hand side converges at once (src/krylov.cpp:26-30)
    op = lambda X: X @ A.T
    pc = lambda X: X * Dinv
    for use_pc in (None, pc):
        res = hs.gmres(op, use_pc, B, tol=1e-10, maxit=80)
        for r in range(3):
            ro = O.gmres(lambda v: A @ v, (lambda v: v) if use_pc is None else (lambda v: Dinv * v), B[r].copy(), 1e-10, 80)
            assert res[r].iterations == ro.iterations and res[r].converged == ro.converged
            np.testing.assert_allclose(res[r].history, ro.history, rtol=1e-9, atol=1e-14)
            if r < 2:
                assert rel(res[r].x, np.linalg.solve(A, B[r])) <= 1e-8
                assert res[r].true_residual <= 1e-9
    few = hs.gmres(op, None, B[0], tol=1e-12, maxit=5, restart=5)  # stops at maxit, not converged
    assert few.iterations == 5 and not few.converged and len(few.history) == 6
    with pytest.raises(ValueError):  # a failing callback aborts the solve (HS_ERR_DATA); its own exception is re-raised
        hs.gmres(lambda X: X[:, :-1], None, B[0])
    z = golden("gmres_2d")
    med = ast.literal_eval(str(z["medium"]))
    s = hs.DdmSolver(hs.ProblemSetup(2, [int(z["n"])] * 2, list(z["parts"]), hs.Medium("constant", kappa=med["media.kappa"]),
                                     pml_width=int(z["pad"])))
    wired = s.gmres(z["b"], float(z["tol"]), int(z["maxit"]), 1)
    seam = hs.gmres(lambda X: s.apply_op(X), lambda X: s.ddm_solve(X, 1, None, False), z["b"], float(z["tol"]),
                    int(z["maxit"]))
    assert seam.iterations == wired.iterations and abs(seam.iterations - int(z["iterations"])) <= 1
    np.testing.assert_allclose(seam.history, wired.history, rtol=1e-8)
    assert rel(seam.x, wired.x) <= 1e-9 and rel(seam.x, z["x"]) <= 1e-7


def test_gmres_restarted(hs, golden):
    z = golden("gmres_2d")
    med = ast.literal_eval(str(z["medium"]))
    s = hs.DdmSolver(hs.ProblemSetup(2, [int(z["n"])] * 2, list(z["parts"]), hs.Medium("constant", kappa=med["media.kappa"]),
                                     pml_width=int(z["pad"])))
    full = s.gmres(z["b"], float(z["tol"]), int(z["maxit"]), 1)
    # a restart length the iteration count never reaches is the reference's full GMRES, bit for bit
    same = s.gmres(z["b"], float(z["tol"]), int(z["maxit"]), 1, restart=full.iterations + 1)
    assert np.array_equal(same.x, full.x) and same.history == full.history
    # GMRES(2): restarts from the current iterate still reach the tolerance
    g2 = s.gmres(z["b"], float(z["tol"]), 200, 1, restart=2)
    assert g2.converged and g2.iterations >= full.iterations
    assert g2.true_residual <= 1e-7 and rel(g2.x, z["x"]) <= 1e-6
    assert len(g2.history) == g2.iterations + 1


def test_apply_op_matches_oracle(hs, golden):
    z = golden("ddm_2d_layered")
    s = hs.DdmSolver(_setup(hs, z))
    so = O.DdmSolver(O.ProblemSetup(O.Box(2), [int(z["n"])] * 2 + [1], list(z["parts"]) + [1],
                                    O.Medium("two_layered", kappa_down=12 * math.pi, kappa_up=8 * math.pi, axis=1,
                                             eta=0.5 + 1 / 128, eps=0.0), O.PmlSpec(width=int(z["pad"]))), factor=False)
    x = z["u"][0]
    assert rel(s.apply_op(x), so.global_op().apply(x)) <= 1e-14


def test_c2_subdomain_factor_against_oracle(hs):
    """One subdomain of BASELINE config 2 (1024^2, 8x8, PML 32, omega = 2 pi 64; 193^2 local
    grid, all four symbolic classes) factorized on the GPU vs the numpy restatement."""
    n, pad, kap = 1024, 32, 2 * math.pi * 64
    so = O.DdmSolver(O.ProblemSetup(O.Box(2), [n, n, 1], [8, 8, 1], O.Medium("constant", kappa=kap),
                                    O.PmlSpec(width=pad)), factor=False)
    g = np.random.default_rng(5)
    for sid in (0, 1, 8, 9):
        st = so.states[sid]
        op = hs.SparseOperator(2, st.grid.range.lo, st.grid.range.hi, st.op.row_ptr, st.op.col, st.op.val)
        f = hs.factorize(op)
        fo = O.factorize(st.op, 2, st.grid.range)
        assert f.stats().factor_nnz == fo.factor_nnz
        b = g.standard_normal((3, st.op.n)) + 1j * g.standard_normal((3, st.op.n))
        X = f.solve(b)
        for r in range(3):
            assert rel(X[r], fo.solve(b[r])) <= 1e-11


@pytest.mark.parametrize("name,rounds,segs", [("ddm_2d_3x2_r2", 1, None), ("ddm_2d_3x2_r2", 2, None),
                                               ("ddm_2d_3x2_r2", 1, 3), ("ddm_2d_2x2", 1, 5),
                                               ("ddm_3d_2x2x2", 1, None), ("ddm_3d_2x2x2", 1, 2)])
def test_streamed_host_path_equals_device_path(hs, golden, monkeypatch, name, rounds, segs):
    """hs_ddm_solve with pinned host buffers streams b in by tiles (stripe x fastest-axis
    segment, in the order the sweep-1 sources read them) and u out by tiles / stripes around the
    macro-step schedule; it must return exactly the device-buffer result (and the pageable-buffer
    one). segs forces the number of fastest-axis segments (HS_TILE_SEGS), so the multi-segment
    tiling is exercised at golden sizes too; 1 round also checks the result against the reference."""
    torch = pytest.importorskip("torch")
    if segs is not None:
        monkeypatch.setenv("HS_TILE_SEGS", str(segs))
    z = golden(name)
    s = hs.DdmSolver(_setup(hs, z))
    b = np.ascontiguousarray(z["b"], dtype=np.complex128)  # (R, N) RHS-major
    R = b.shape[0]
    hb = torch.from_numpy(b.view(np.float64)).pin_memory()
    hu = torch.empty_like(hb).pin_memory()
    s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), R, rounds, True)
    db = hb.cuda()
    du = torch.empty_like(db)
    s.ddm_solve_device(db.data_ptr(), du.data_ptr(), R, rounds, True)
    torch.cuda.synchronize()
    assert torch.equal(hu, du.cpu())
    u_pageable = s.ddm_solve(b, rounds, None, True)
    uh = hu.numpy().view(np.complex128).reshape(R, -1)
    assert np.array_equal(uh, np.asarray(u_pageable).reshape(R, -1))
    if rounds == int(z["rounds"]):
        for r in range(R):
            assert rel(uh[r], z["u"][r]) <= 1e-9


def test_global_direct_solve_matches_sparse_lu(hs):
    """global_direct_solve (src/harness.cpp:185-214) on the device factorization against an
    independent sparse LU (SuperLU) of the same J-scaled global operator; and the DDM solution
    compared with it, as the reference's direct-solver mode does (compare.global)."""
    spla = pytest.importorskip("scipy.sparse.linalg")
    sp = pytest.importorskip("scipy.sparse")
    n, pad, kap = 128, 12, 2 * math.pi * 8
    so = O.DdmSolver(O.ProblemSetup(O.Box(2), [n, n, 1], [2, 2, 1], O.Medium("constant", kappa=kap),
                                    O.PmlSpec(width=pad)))
    f = O.gaussian_source(so.ggrid, O.Box(2), [[0.5, 0.5], [0.3, 0.62]], 2.0 / n).T.copy()  # (2, N)
    s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [2, 2], hs.Medium("constant", kappa=kap), pml_width=pad))
    stats = []
    u = s.global_direct_solve(f, stats)
    op = so.global_op()
    A = sp.csr_matrix((op.val, op.col, op.row_ptr), shape=(len(op.row_ptr) - 1,) * 2).tocsc()
    b = so.scale_source(f.T).T.copy()
    lu = spla.splu(A)
    for r in range(2):
        assert rel(u[r], lu.solve(b[r])) <= TOL
    assert stats[0].n == A.shape[0] and stats[0].matrix_nnz == A.nnz
    U = s.ddm_solve(b, 1)
    for r in range(2):  # sanity: one round of diagonal sweeps approximates the global solve
        assert rel(U[r], u[r]) < 0.5


def test_3d_moderate_against_oracle(hs):
    """3D at a size with real fronts (32^3 grid, 2x2x2 subdomains of 29^3 nodes, separators up to
    29^2): batched device sweeps against the numpy restatement, counters bit-exact."""
    n, pad, kap = 32, 6, 2 * math.pi * 3
    so = O.DdmSolver(O.ProblemSetup(O.Box(3), [n, n, n], [2, 2, 2], O.Medium("constant", kappa=kap),
                                    O.PmlSpec(width=pad)))
    f = O.gaussian_source(so.ggrid, O.Box(3), [[0.5, 0.5, 0.5], [0.3, 0.6, 0.45]], 2.0 / n)
    b = so.scale_source(f).T.copy()
    s = hs.DdmSolver(hs.ProblemSetup(3, [n] * 3, [2, 2, 2], hs.Medium("constant", kappa=kap), pml_width=pad))
    reps = []
    U = s.ddm_solve(b, 1, reps, True)
    for r in range(2):
        uo, ro = so.ddm_solve(b[r].copy(), 1, True)
        assert rel(U[r], uo) <= TOL
        assert [getattr(reps[r], k) for k in COUNTERS] == [getattr(ro, k) for k in COUNTERS]
    # large fronts are factorized by CTA clusters: an independent factorization is bitwise equal
    s2 = hs.DdmSolver(hs.ProblemSetup(3, [n] * 3, [2, 2, 2], hs.Medium("constant", kappa=kap), pml_width=pad))
    assert np.array_equal(s2.ddm_solve(b, 1), U)


@pytest.mark.parametrize("dim", [2, 3])
def test_cluster_factorization_path_against_oracle(hs, monkeypatch, dim):
    """The blocked cluster factorization (hs_factor.cu) forced onto every front with m >= 96
    (HS_FACTOR_BIG_M): 2D C1-size subdomains (105^2, fronts up to m = 157) and 3D 2x2x2 (fronts
    up to m ~ 500, several 64-row blocks and partial panels) against the numpy restatement."""
    monkeypatch.setenv("HS_FACTOR_BIG_M", "96")
    if dim == 2:
        n, pad, kap, parts = 256, 20, 2 * math.pi * 16, [4, 4]
        centers = [[0.5, 0.5], [0.3125, 0.6]]
    else:
        n, pad, kap, parts = 24, 5, 2 * math.pi * 2, [2, 2, 2]
        centers = [[0.5, 0.5, 0.5], [0.3, 0.6, 0.45]]
    so = O.DdmSolver(O.ProblemSetup(O.Box(dim), [n] * dim + [1] * (3 - dim), parts + [1] * (3 - dim),
                                    O.Medium("constant", kappa=kap), O.PmlSpec(width=pad)))
    b = so.scale_source(O.gaussian_source(so.ggrid, O.Box(dim), centers, 2.0 / n)).T.copy()
    s = hs.DdmSolver(hs.ProblemSetup(dim, [n] * dim, parts, hs.Medium("constant", kappa=kap), pml_width=pad))
    reps = []
    U = s.ddm_solve(b, 1, reps, True)
    for r in range(2):
        uo, ro = so.ddm_solve(b[r].copy(), 1, True)
        assert rel(U[r], uo) <= TOL
        assert [getattr(reps[r], k) for k in COUNTERS] == [getattr(ro, k) for k in COUNTERS]
    s2 = hs.DdmSolver(hs.ProblemSetup(dim, [n] * dim, parts, hs.Medium("constant", kappa=kap), pml_width=pad))
    assert np.array_equal(s2.ddm_solve(b, 1), U)  # the cluster factorization is deterministic


def test_gridded_medium_against_reference(hs, tmp_path):
    """BASELINE config 4's medium kind at small scale: a seeded smooth velocity grid (HSVG file
    for the reference, the same samples for the device), one DDM application and GMRES against
    oracle/_ref (the reference compiled in place) on the same inputs."""
    from oracle import ref
    from paper_2003_02585_b200 import sources
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    nl, n, pad, omega = 64, 64, 8, 2 * math.pi * 4
    c = sources.gaussian_random_velocity(nl, 7, corr_len=0.1)
    path = str(tmp_path / "v.hsvg")
    hs.write_velocity_grid(path, hs.VelocityGrid(2, [nl + 1, nl + 1, 1], [0.0, 0.0, 0.0], [1 / nl, 1 / nl, 0.0], c.ravel()))
    med = hs.Medium("gridded", velocity=c.ravel(), vel_n=(nl + 1, nl + 1, 1), vel_origin=(0.0, 0.0, 0.0),
                    vel_spacing=(1 / nl, 1 / nl, 0.0), omega=omega)
    s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [2, 2], med, pml_width=pad))
    r = ref.RefSolver({"dim": 2, "grid.n": [n, n], "partition": [2, 2], "pml.width": pad, "media.kind": "gridded",
                       "media.velocity_file": path, "media.omega": omega}, 4)
    f = sources.gaussian_sources(2, s.lo, s.hi, [1 / n] * 2, [0.0, 0.0], [[0.3, 0.4], [0.7, 0.2]], 2.0 / n)
    b = s.scale_source(f)
    assert np.array_equal(b[0], r.scale_source(f[0]))
    reps = []
    U = s.ddm_solve(b, 1, reps, True)
    for i in range(2):
        u0, rep0 = r.ddm_solve(b[i], 1, True)
        assert rel(U[i], u0) <= TOL
        assert [getattr(reps[i], k) for k in COUNTERS] == [rep0[k] for k in COUNTERS]
    g = s.gmres(b[0], 1e-8, 60, 1)
    xr, gr = r.gmres(b[0], 1e-8, 60, 1)
    assert abs(g.iterations - gr["iterations"]) <= 1 and rel(g.x, xr) <= 1e-7


def test_batches_beyond_the_device_batch_and_zero_rhs(hs, golden):
    """nrhs above the 64-RHS device batch (two batches) equals per-RHS solves (to roundoff: the
    split-K shape of the critical path follows the batch width) and the reference; an all-zero RHS
    gives an exactly zero field with every task skipped (src/sweeper.cpp:240-251)."""
    z = golden("ddm_2d_2x2")
    s = hs.DdmSolver(_setup(hs, z))
    rng = np.random.default_rng(5)
    B = np.repeat(z["b"], 35, axis=0) * (1.0 + 0.25 * rng.standard_normal((70, 1)))
    B[69] = 0.0
    reps = []
    U = s.ddm_solve(B, 1, reps, True)
    for r in (0, 31, 32, 63, 64, 68):
        assert rel(U[r], s.ddm_solve(B[r], 1)) <= 1e-12
    assert not np.any(U[69])
    assert reps[69].local_solves == 0 and reps[69].skipped_zero_solves == 4 * s.nsub


@pytest.mark.parametrize("dim,n,parts,pad,rounds", [(2, [64, 40], [4, 2], 6, 3), (3, [24, 16, 16], [3, 2, 1], 4, 1),
                                                    (2, [36, 36], [1, 3], 5, 2)])
def test_anisotropic_grids_against_reference(hs, dim, n, parts, pad, rounds):
    """Non-square grids, unequal and unit partition counts, 2-3 rounds: the device path against
    oracle/_ref (the reference compiled in place) on the same seeded sources, u <= 1e-9 and the
    counters exact."""
    from oracle import ref
    from paper_2003_02585_b200 import sources
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    kap = 2 * math.pi * 3
    s = hs.DdmSolver(hs.ProblemSetup(dim, n, parts, hs.Medium("constant", kappa=kap), pml_width=pad))
    r = ref.RefSolver({"dim": dim, "grid.n": n, "partition": parts, "pml.width": pad, "media.kind": "constant",
                       "media.kappa": kap}, 4)
    assert r.N == s.global_n
    f = sources.gaussian_sources(dim, s.lo, s.hi, [1.0 / x for x in n], [0.0] * 3,
                                 sources.seeded_centers(11, 2, dim), 2.0 / max(n))
    b = s.scale_source(f)
    reps = []
    U = s.ddm_solve(b, rounds, reps, True)
    for i in range(2):
        assert np.array_equal(b[i], r.scale_source(f[i]))
        u0, rep0 = r.ddm_solve(b[i], rounds, True)
        assert rel(U[i], u0) <= TOL
        assert [getattr(reps[i], k) for k in COUNTERS] == [rep0[k] for k in COUNTERS]
        np.testing.assert_allclose(reps[i].round_residuals, rep0["round_residuals"], rtol=1e-6)


@pytest.mark.parametrize("rounds", [2, 3])
def test_sparse_sources_wide_batch_against_reference(hs, rounds):
    """A ragged wide batch of compactly supported sources scattered over the subdomains, some
    columns exactly zero: most (task, RHS) pairs are exact-zero solves, which the reference skips
    one by one (src/sweeper.cpp:240-251). The device orders the columns by source location, skips
    the RHS groups that are all zero for a task and narrows half-zero groups; every column and its
    report (mapped back through the column order) must equal the reference's for that source.
    Two rounds run the fused accumulate, three (12 sweeps > 8 x buffers) the per-sweep one."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    n, parts, pad = [64, 64], [4, 4], 6
    kap = 2 * math.pi * 4
    s = hs.DdmSolver(hs.ProblemSetup(2, n, parts, hs.Medium("constant", kappa=kap), pml_width=pad))
    r = ref.RefSolver({"dim": 2, "grid.n": n, "partition": parts, "pml.width": pad, "media.kind": "constant",
                       "media.kappa": kap}, 4)
    gx = s.hi[0] - s.lo[0] + 1
    rng = np.random.default_rng(23)
    R = 41
    B = np.zeros((R, s.global_n), complex)
    for c in range(R):
        if c % 7 == 3:
            continue  # an all-zero column
        ix, iy = rng.integers(2, n[0] - 2), rng.integers(2, n[1] - 2)
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                B[c, (ix + dx - s.lo[0]) + gx * (iy + dy - s.lo[1])] = rng.standard_normal() + 1j * rng.standard_normal()
    reps = []
    U = s.ddm_solve(B, rounds, reps, True)
    for c in (0, 3, 5, 16, 17, 24, 31, 33, 40):
        u0, rep0 = r.ddm_solve(B[c], rounds, True)
        if not np.any(B[c]):
            assert not np.any(U[c]) and reps[c].local_solves == 0
            continue
        assert rel(U[c], u0) <= TOL
        assert [getattr(reps[c], k) for k in COUNTERS] == [rep0[k] for k in COUNTERS]
        assert reps[c].skipped_zero_solves > 0
        np.testing.assert_allclose(reps[c].round_residuals, rep0["round_residuals"], rtol=1e-6)
    # the streamed host-buffer path (its own column order, from samples of the host buffer)
    import torch
    hb = torch.from_numpy(B.view(np.float64)).pin_memory()
    hu = torch.empty_like(hb).pin_memory()
    s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), R, rounds, True)
    Uh = hu.numpy().view(np.complex128)
    for c in range(R):  # (32 + 9 RHS batches there, one 41-RHS batch above: equal to roundoff)
        assert (rel(Uh[c], U[c]) <= 1e-12) if np.any(B[c]) else not np.any(Uh[c])


_ALT_SCRIPT = r"""
import ast, os, sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2003_02585_b200 as hs
worst = 0.0
for name in ["ddm_2d_3x2_r2", "ddm_3d_2x2x2", "ddm_2d_layered"]:
    z = np.load({root!r} + "/tests/golden/" + name + ".npz")
    med = ast.literal_eval(str(z["medium"]))
    if med["media.kind"] == "constant":
        m = hs.Medium("constant", kappa=med["media.kappa"])
    else:
        m = hs.Medium("two_layered", kappa_down=med["media.kappa_down"], kappa_up=med["media.kappa_up"],
                      axis=med["media.axis"], eta=med["media.eta_L"], eps=med["media.epsilon"])
    dim = int(z["dim"])
    s = hs.DdmSolver(hs.ProblemSetup(dim, [int(z["n"])] * dim, list(z["parts"]), m, pml_width=int(z["pad"])))
    rep = int(os.environ.get("HS_ALT_REPEAT", "1"))  # the fixture's RHS repeated (a wider batch)
    n0 = z["b"].shape[0]
    U = s.ddm_solve(np.tile(z["b"], (rep, 1)), int(z["rounds"]), None, True)
    for r in range(U.shape[0]):
        worst = max(worst, float(np.linalg.norm(U[r] - z["u"][r % n0]) / np.linalg.norm(z["u"][r % n0])))
print("WORST", worst)
"""


@pytest.mark.parametrize("env", [{"HS_M3": "0"}, {"HS_GRAPH": "0"}, {"HS_ORDER": "0", "HS_MAX_CHUNKS": "1"},
                                 {"HS_QUAD": "1", "HS_ALT_REPEAT": "7"}, {"HS_ALT_REPEAT": "9"},
                                 {"HS_NO_GROUP_SKIP": "1", "HS_NO_RHS_SORT": "1", "HS_ALT_REPEAT": "9"}])
def test_alternate_engine_paths_match_reference(env):
    """The engine's alternates, each selected per process by an environment switch, against the
    reference's golden u: the four-product solve kernels (HS_M3=0, 4 CTAs/SM), stream-by-stream
    launches instead of the captured CUDA graph (HS_GRAPH=0), and the plain level order with
    the widest split-K chunks (HS_ORDER=0, HS_MAX_CHUNKS=1: 16-block chunks; a band
    longer than 16 blocks still splits), the quad dequeue (HS_QUAD=1: one CTA takes the RHS groups of
    a band chunk together, lists padded with null items; the fixture's RHS repeated to a ragged wide
    batch), and a ragged wide batch on the default path (odd RHS count: the fused accumulate's RHS
    pairs, partial last RHS group)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _ALT_SCRIPT.format(root=root)], capture_output=True, text=True,
                       env={**os.environ, **env}, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    worst = float(r.stdout.split("WORST")[-1])
    assert worst <= TOL


def test_concurrent_solves_on_one_factorization(hs, golden):
    """Factorization::solve is "reentrant; safe for concurrent calls on one factorization"
    (include/helmsweep/direct.hpp:29): two host threads solving different right-hand sides on one
    handle (ctypes releases the GIL) each get exactly the single-threaded result."""
    import threading
    z = golden("direct_3d")
    f = hs.factorize(sparse_op(hs, z))
    n = f.stats().n
    g = np.random.default_rng(29)
    B = [g.standard_normal((3, n)) + 1j * g.standard_normal((3, n)) for _ in range(4)]
    want = [f.solve(b) for b in B]
    got = [None] * len(B)
    errs = []

    def work(i):
        try:
            for _ in range(5):
                got[i] = f.solve(B[i])
                if not np.array_equal(got[i], want[i]):
                    errs.append(i)
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(B))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs


def test_null_stream_is_ordered_after_legacy_default_stream(hs, golden):
    """stream = NULL means the legacy default stream (include/helmsweep_b200.h): b written there by
    a kernel, with no host synchronisation, must be read only after that kernel (the solver's own
    stream is non-blocking). Checked for hs_ddm_solve_device and hs_factor_solve_device."""
    torch = pytest.importorskip("torch")
    z = golden("ddm_2d_3x2_r2")
    s = hs.DdmSolver(_setup(hs, z))
    b = np.ascontiguousarray(z["b"], dtype=np.complex128)
    R = b.shape[0]
    rounds = int(z["rounds"])
    want = s.ddm_solve(b, rounds, None, False)
    src = torch.from_numpy(b.view(np.float64)).cuda()
    torch.cuda.synchronize()
    with torch.cuda.stream(torch.cuda.default_stream()):
        db = torch.zeros_like(src)
        du = torch.zeros_like(src)
        big = torch.ones(64 << 20, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        for _ in range(20):  # keep the legacy stream busy before b gets its values
            big.mul_(1.0000001)
        db.copy_(src)
        s.ddm_solve_device(db.data_ptr(), du.data_ptr(), R, rounds, False, 0)
    torch.cuda.synchronize()
    got = du.cpu().numpy().view(np.complex128).reshape(R, -1)
    assert np.array_equal(got, np.asarray(want).reshape(R, -1))
    zf = golden("direct_2d")
    f = hs.factorize(sparse_op(hs, zf))
    xb = torch.from_numpy(np.ascontiguousarray(zf["b"], dtype=np.complex128).view(np.float64)).cuda()
    torch.cuda.synchronize()
    dx = torch.zeros_like(xb)
    for _ in range(20):
        big.mul_(1.0000001)
    dx.copy_(xb)
    f.solve_device(dx.data_ptr(), 1, 0)
    torch.cuda.synchronize()
    assert rel(dx.cpu().numpy().view(np.complex128), zf["x"]) <= 1e-12
