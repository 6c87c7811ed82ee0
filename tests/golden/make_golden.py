"""Generates the golden fixtures in tests/golden/ by running the REFERENCE itself
(oracle/_ref/libhelmsweep_ref.so, compiled in place from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are small .npz files; GPU boxes only read them.

Cases (every input is seeded; sources follow SURVEY.md §8(d): f = exp(-|x-xs|^2/(2 sigma^2)),
sigma = 2h, on interior nodes, b = DdmSolver::scale_source(f) computed by the reference):
  direct_2d / direct_3d   tests/test_direct.cpp:95-104 operators, reference solve of seeded b
  ddm_*                   DdmSolver::ddm_solve u, SolveReport counters, contrib norms, residuals
  gmres_2d                run_precond-style GMRES: iterations, history, x
  routing                 route_trace tables (Appendix B of SURVEY.md)
  io_*                    HSVG velocity grids and an HSFD field dump written by the reference's own
                          write_velocity_grid / write_field (byte-exact format pins)
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import hs_oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

COUNTERS = ["traces_generated", "traces_routed", "traces_discarded", "local_solves", "skipped_zero_solves"]

DDM_CASES = {
    # name: (dim, n, parts, pad, medium-dict, rounds, centers)
    "ddm_2d_2x2": (2, 48, (2, 2), 10, {"media.kind": "constant", "media.kappa": 10 * math.pi}, 1,
                   [[0.3, 0.3], [0.71, 0.62]]),
    "ddm_2d_3x2_r2": (2, 48, (3, 2), 8, {"media.kind": "constant", "media.kappa": 9 * math.pi}, 2,
                      [[0.5, 0.5], [0.2, 0.81]]),
    "ddm_2d_layered": (2, 64, (4, 4), 8,
                       {"media.kind": "two_layered", "media.kappa_down": 12 * math.pi,
                        "media.kappa_up": 8 * math.pi, "media.axis": 1,
                        "media.eta_L": 0.5 + 1 / 128, "media.epsilon": 0.0}, 2,
                       [[0.37, 0.41], [0.66, 0.7]]),
    "ddm_3d_2x2x2": (3, 16, (2, 2, 2), 4, {"media.kind": "constant", "media.kappa": 8.0}, 1,
                     [[0.3, 0.6, 0.45]]),
}


def cfg(dim, n, parts, pad, med, extra=None):
    d = {"dim": dim, "grid.n": [n] * dim, "partition": list(parts), "pml.width": pad}
    d.update(med)
    if extra:
        d.update(extra)
    return d


def make_ddm(name, dim, n, parts, pad, med, rounds, centers):
    s = R.RefSolver(cfg(dim, n, parts, pad, med), 1)
    ggrid = O.LocalGrid(dim, O.GridRange(dim, s.lo, s.hi), s.hgrid, s.origin)
    interior = O.Box(dim, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    f = O.gaussian_source(ggrid, interior, centers, 2.0 / n)
    out = {"dim": dim, "n": n, "parts": np.array(parts), "pad": pad, "rounds": rounds,
           "centers": np.array(centers), "medium": repr(med)}
    B, U, C, N, RR = [], [], [], [], []
    for r in range(f.shape[1]):
        b = s.scale_source(f[:, r].copy())
        u, rep = s.ddm_solve(b, rounds, True)
        B.append(b)
        U.append(u)
        C.append([rep[k] for k in COUNTERS])
        N.append(rep["sweep_contrib_norm"])
        RR.append(rep["round_residuals"])
    out.update(b=np.array(B), u=np.array(U), counters=np.array(C), contrib_norm=np.array(N),
               round_residuals=np.array(RR))
    out["factor_nnz"] = np.array([s.sub_info(i)["factor_nnz"] for i in range(s.nsub)])
    out["peak_bytes"] = np.array([s.sub_info(i)["peak_bytes"] for i in range(s.nsub)])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def make_direct(name, dim, n, pad, kappa, seed):
    rp, col, val = R.pml_operator(dim, n, pad, kappa)
    lo = [-pad] * dim + [0] * (3 - dim)
    hi = [n + pad] * dim + [0] * (3 - dim)
    f = R.RefFactorization(dim, lo, hi, rp, col, val)
    rng = np.random.default_rng(seed)
    b = rng.uniform(-1, 1, f.n) + 1j * rng.uniform(-1, 1, f.n)
    x = f.solve(b)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), dim=dim, n=n, pad=pad, kappa=kappa,
                        row_ptr=rp, col=col, val=val, lo=np.array(lo), hi=np.array(hi), b=b, x=x,
                        factor_nnz=f.factor_nnz)


def make_gmres():
    dim, n, parts, pad = 2, 48, (4, 4), 10
    med = {"media.kind": "constant", "media.kappa": 10 * math.pi}
    s = R.RefSolver(cfg(dim, n, parts, pad, med), 1)
    ggrid = O.LocalGrid(dim, O.GridRange(dim, s.lo, s.hi), s.hgrid, s.origin)
    f = O.gaussian_source(ggrid, O.Box(2, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)), [[0.31, 0.29]], 2.0 / n)
    b = s.scale_source(f[:, 0].copy())
    x, info = s.gmres(b, 1e-8, 60, 1)
    np.savez_compressed(os.path.join(HERE, "gmres_2d.npz"), dim=dim, n=n, parts=np.array(parts), pad=pad,
                        medium=repr(med), b=b, x=x, iterations=info["iterations"],
                        history=np.array(info["history"]), true_residual=info["true_residual"],
                        tol=1e-8, maxit=60)


def make_routing():
    out = {}
    for dim in (2, 3):
        for rounds in (1, 2):
            nl = rounds * (1 << dim)
            tab = np.zeros((nl, 2 * dim), dtype=np.int64)
            for l in range(1, nl + 1):
                for d in range(2 * dim):
                    tab[l - 1, d] = R.route(dim, rounds, l, d // 2, 1 if d & 1 else -1)
            out[f"route_{dim}d_r{rounds}"] = tab
    np.savez_compressed(os.path.join(HERE, "routing.npz"), **out)


def make_io():
    """HSVG / HSFD files written by the reference (include/helmsweep/media.hpp:22-27,
    src/harness.cpp:32-53) plus the arrays they hold."""
    import ctypes
    L = R.lib()
    rng = np.random.default_rng(7)
    dbl3, int3 = ctypes.c_double * 3, ctypes.c_int * 3
    arrays = {}
    for name, dim, n, org, sp in [("io_vel2d", 2, [5, 4, 1], [0.0, -0.5, 0.0], [0.25, 0.5, 0.0]),
                                  ("io_vel3d", 3, [3, 3, 2], [0.1, 0.2, 0.3], [0.5, 0.5, 1.0])]:
        c = (1.0 + rng.random(int(np.prod(n[:dim])))).astype(np.float32)
        path = os.path.join(HERE, name + ".hsvg")
        rc = L.hsref_write_velocity_grid(path.encode(), dim, int3(*n), dbl3(*org), dbl3(*sp),
                                         c.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        assert rc == 0, L.hsref_last_error()
        arrays[name] = c
        arrays[name + "_hdr"] = np.array([dim, *n], dtype=np.int64)
        arrays[name + "_geo"] = np.array([*org, *sp], dtype=np.float64)
    lo, hi, h, org = [-2, -1, 0], [3, 3, 0], [0.125, 0.25, 0.0], [0.0, 0.0, 0.0]
    u = (rng.standard_normal(6 * 5) + 1j * rng.standard_normal(6 * 5)).astype(np.complex128)
    path = os.path.join(HERE, "io_field2d.hsfd")
    rc = L.hsref_write_field(path.encode(), 2, int3(*lo), int3(*hi), dbl3(*h), dbl3(*org),
                             u.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert rc == 0, L.hsref_last_error()
    arrays["io_field2d"] = u
    arrays["io_field2d_geo"] = np.array([*lo, *hi], dtype=np.int64)
    arrays["io_field2d_hdr"] = np.array([*h, *org], dtype=np.float64)
    np.savez(os.path.join(HERE, "io.npz"), **arrays)


if __name__ == "__main__":
    if sys.argv[1:] == ["io"]:
        make_io()
        sys.exit(0)
    make_io()
    make_routing()
    make_direct("direct_2d", 2, 12, 3, 9.0, 11)
    make_direct("direct_3d", 3, 8, 3, 9.0, 11)
    make_direct("direct_2d_16", 2, 16, 4, 11.0, 33)
    for k, v in DDM_CASES.items():
        make_ddm(k, *v)
    make_gmres()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
