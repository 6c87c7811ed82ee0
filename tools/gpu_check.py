"""Developer diagnostic: runs the GPU path against the numpy oracle on small cases and
prints errors (no asserts) so one GPU call reports every mismatch at once."""
import math, sys, time, traceback
import numpy as np
sys.path.insert(0, '.')
import paper_2003_02585_b200 as hs
from oracle import hs_oracle as O

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

def run(name, fn):
    t = time.time()
    try:
        fn()
        print(f"[ok] {name} ({time.time()-t:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()

def fact_tests():
    # pml operator 2D 12^2 pad 3 kappa 9 (tests/test_direct.cpp:95-104)
    for dim, n in ((2, 12), (3, 8)):
        pad = 3
        g = O.LocalGrid(dim, O.GridRange(dim, [-pad]*dim + [0]*(3-dim), [n+pad]*dim + [0]*(3-dim)), [1.0/n]*dim + [0.0]*(3-dim), [0.0]*3)
        c = O.PmlCoefficients(O.PmlSpec(width=pad), O.Box(dim, (0.,0.,0.), (1.,1.,1.)), g)
        op = O.assemble(g, c, np.full(g.node_count(), 9.0))
        F = hs.factorize(hs.SparseOperator(dim, g.range.lo, g.range.hi, op.row_ptr, op.col, op.val))
        fo = O.factorize(op, dim, g.range)
        rng = np.random.default_rng(11)
        b = rng.uniform(-1, 1, op.n) + 1j * rng.uniform(-1, 1, op.n)
        x = F.solve(b)
        xo = fo.solve(b)
        res = np.linalg.norm(op.apply(x) - b) / np.linalg.norm(b)
        print(f"  dim{dim}: resid {res:.3e} vs-oracle {rel(x, xo):.3e} nnz {F.stats().factor_nnz} {fo.factor_nnz} peak {F.stats().peak_bytes} {fo.peak_bytes}")
        B = np.stack([b, 2*b, rng.uniform(-1,1,op.n)+0j, np.zeros(op.n, complex), b*1j])
        X = F.solve(B)
        print("  batch vs single:", [rel(X[i], F.solve(B[i])) if np.any(B[i]) else float(np.abs(X[i]).max()) for i in range(5)])
        x2 = F.solve(b)
        print("  bitwise repeat:", np.array_equal(x, x2))
    # 1x1 and singular
    op1 = hs.SparseOperator(2, [0,0,0], [0,0,0], np.array([0,1]), np.array([0]), np.array([2.0+0j]))
    print("  1x1:", hs.factorize(op1).solve(np.array([3+1j])))
    opd = hs.SparseOperator(2, [0,0,0], [2,0,0], np.array([0,1,2,3]), np.array([0,1,2]), np.array([1.0,0.0,1.0])+0j)
    try:
        hs.factorize(opd); print("  singular NOT raised")
    except hs.SingularMatrixError as e:
        print("  singular pivot_index", e.pivot_index)

def ddm_case(n, parts, pad, kappa, rounds=1, R=1, dim=2, centers=None):
    setup_o = O.ProblemSetup(O.Box(dim,(0.,0.,0.),(1.,1.,1.)), [n]*dim+[1]*(3-dim), list(parts)+[1]*(3-dim), O.Medium('constant', kappa=kappa), O.PmlSpec(width=pad))
    so = O.DdmSolver(setup_o)
    setup = hs.ProblemSetup(dim, [n]*dim, list(parts), hs.Medium('constant', kappa=kappa), pml_width=pad)
    t = time.time(); s = hs.DdmSolver(setup); print(f"  gpu setup+factor {time.time()-t:.2f}s (factor_seconds {s.factor_seconds():.3f})")
    for sid in range(len(so.states)):
        st = s.sub_stats(sid)
        if st.factor_nnz != so.states[sid].fact.factor_nnz: print("  factor_nnz mismatch sub", sid)
    if centers is None:
        centers = O.seeded_centers(7, R, O.Box(dim,(0.,0.,0.),(1.,1.,1.)))
    f = O.gaussian_source(so.ggrid, O.Box(dim,(0.,0.,0.),(1.,1.,1.)), centers, 2.0/n)
    b = so.scale_source(f)  # (N, R)
    reps = []
    t = time.time(); U = s.ddm_solve(b.T.copy(), rounds, reps, True); tg = time.time()-t
    for r in range(R):
        uo, ro = so.ddm_solve(b[:, r].copy(), rounds, True)
        g = reps[r]
        cnt_ok = all(getattr(ro,k)==getattr(g,k) for k in ['traces_generated','traces_routed','traces_discarded','local_solves','skipped_zero_solves'])
        print(f"  rhs{r}: rel {rel(U[r], uo):.3e} counters {'OK' if cnt_ok else 'MISMATCH'} gpu=({g.local_solves},{g.skipped_zero_solves},{g.traces_routed},{g.traces_discarded}) ref=({ro.local_solves},{ro.skipped_zero_solves},{ro.traces_routed},{ro.traces_discarded}) norms {np.max(np.abs(np.array(g.sweep_contrib_norm)-np.array(ro.sweep_contrib_norm))/np.array(ro.sweep_contrib_norm).max()):.2e} res {g.round_residuals} {ro.round_residuals}")
    print(f"  gpu ddm time {tg:.3f}s, sweep total {reps[0].sweep_seconds_total:.4f}s")
    return s, so, b

def gmres_case():
    n, parts, pad, kappa = 48, (2, 2), 10, 10*math.pi
    s, so, b = ddm_case(n, parts, pad, kappa, 1, 1, centers=[[0.3, 0.3]])
    g = s.gmres(b[:, 0].copy(), 1e-8, 30, 1)
    go = O.gmres(lambda v: so.global_op().apply(v), lambda v: so.ddm_solve(v, 1)[0], b[:, 0].copy(), 1e-8, 30)
    print(f"  gmres iters gpu {g.iterations} ref {go.iterations} true {g.true_residual:.2e} {go.true_residual:.2e} xrel {rel(g.x, go.x):.2e}")
    y = s.apply_op(b[:, 0].copy()); yo = so.global_op().apply(b[:, 0].copy())
    print(f"  apply_op rel {rel(y, yo):.2e}")

print("devices", hs.device_count())
run("factor/solve pins", fact_tests)
run("ddm 64^2 2x2 R=1", lambda: ddm_case(64, (2, 2), 8, 30.0))
run("ddm 64^2 2x2 R=5 rounds=2", lambda: ddm_case(64, (2, 2), 8, 30.0, rounds=2, R=5))
run("ddm 3D 16^3 2x2x2 R=2", lambda: ddm_case(16, (2, 2, 2), 4, 8.0, R=2, dim=3))
run("ddm C1 256^2 4x4 R=1 centre", lambda: ddm_case(256, (4, 4), 20, 2*math.pi*16, centers=[[0.5, 0.5]]))
run("ddm C1 R=16", lambda: ddm_case(256, (4, 4), 20, 2*math.pi*16, R=16))
run("gmres", gmres_case)
