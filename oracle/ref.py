"""ctypes binding of oracle/_ref/libhelmsweep_ref.so (the reference compiled in place).

TEST INFRASTRUCTURE ONLY (tests/, bench.py reference + cpu_baseline legs). See
oracle/ref_driver.cpp for the entry points and the reference API each one calls.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhelmsweep_ref.so")

_c_int_p = ctypes.POINTER(ctypes.c_int)
_c_ll_p = ctypes.POINTER(ctypes.c_longlong)
_c_dbl_p = ctypes.POINTER(ctypes.c_double)


class RefReport(ctypes.Structure):
    _fields_ = [
        ("factor_seconds", ctypes.c_double),
        ("sweep_seconds_total", ctypes.c_double),
        ("median_subdomain_solve_seconds", ctypes.c_double),
        ("traces_generated", ctypes.c_longlong),
        ("traces_routed", ctypes.c_longlong),
        ("traces_discarded", ctypes.c_longlong),
        ("local_solves", ctypes.c_longlong),
        ("skipped_zero_solves", ctypes.c_longlong),
        ("n_sweeps", ctypes.c_int),
        ("n_round_residuals", ctypes.c_int),
    ]


class RefError(RuntimeError):
    def __init__(self, code, msg, pivot=None):
        super().__init__(msg)
        self.code = code
        self.pivot_index = pivot


_lib = None


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.hsref_last_error.restype = ctypes.c_char_p
    return _lib


def _p(a):
    return a.ctypes.data_as(_c_dbl_p)


def _check(rc, pivot=None):
    if rc != 0:
        raise RefError(rc, lib().hsref_last_error().decode(), pivot)


def config_text(d: dict) -> str:
    lines = []
    for k, v in d.items():
        if isinstance(v, (list, tuple)):
            v = " ".join(repr(x) if isinstance(x, float) else str(x) for x in v)
        elif isinstance(v, float):
            v = repr(v)
        lines.append(f"{k} = {v}")
    return "\n".join(lines) + "\n"


class RefSolver:
    """DdmSolver of the reference (src/sweeper.cpp:133-157) built from config keys."""

    def __init__(self, cfg: dict, workers: int = 0):
        L = lib()
        self.h = ctypes.c_void_p()
        _check(L.hsref_solver_create(config_text(cfg).encode(), int(workers), ctypes.byref(self.h)))
        dim, n, ns, fs = ctypes.c_int(), ctypes.c_longlong(), ctypes.c_int(), ctypes.c_double()
        lo, hi = (ctypes.c_int * 3)(), (ctypes.c_int * 3)()
        hh, org = (ctypes.c_double * 3)(), (ctypes.c_double * 3)()
        L.hsref_solver_info(self.h, ctypes.byref(dim), ctypes.byref(n), ctypes.byref(ns),
                            ctypes.byref(fs), lo, hi, hh, org)
        self.dim, self.N, self.nsub, self.factor_seconds = dim.value, n.value, ns.value, fs.value
        self.lo, self.hi, self.hgrid, self.origin = list(lo), list(hi), list(hh), list(org)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.hsref_solver_destroy(self.h)
            self.h = None

    def sample_source(self):
        f = np.zeros(self.N, dtype=np.complex128)
        _check(lib().hsref_sample_source(self.h, _p(f)))
        return f

    def scale_source(self, f):
        f = np.ascontiguousarray(f, dtype=np.complex128)
        b = np.zeros(self.N, dtype=np.complex128)
        _check(lib().hsref_scale_source(self.h, _p(f), _p(b)))
        return b

    def ddm_solve(self, b, rounds=1, track=False):
        b = np.ascontiguousarray(b, dtype=np.complex128)
        u = np.zeros(self.N, dtype=np.complex128)
        rep = RefReport()
        ns = rounds * (1 << self.dim)
        ss = np.zeros(ns)
        cn = np.zeros(ns)
        rr = np.zeros(rounds)
        _check(lib().hsref_ddm_solve(self.h, _p(b), _p(u), int(rounds), int(track), ctypes.byref(rep),
                                     _p(ss), _p(cn), _p(rr)))
        out = {f: getattr(rep, f) for f, _ in RefReport._fields_}
        out["sweep_seconds"] = ss.tolist()
        out["sweep_contrib_norm"] = cn.tolist()
        out["round_residuals"] = rr[: rep.n_round_residuals].tolist()
        return u, out

    def sub_info(self, sub):
        a = [(ctypes.c_int * 3)() for _ in range(4)]
        v = [ctypes.c_longlong() for _ in range(4)]
        lib().hsref_sub_info(self.h, int(sub), *a, *[ctypes.byref(x) for x in v])
        return dict(lo=list(a[0]), hi=list(a[1]), owned_lo=list(a[2]), owned_hi=list(a[3]),
                    n=v[0].value, nnz=v[1].value, factor_nnz=v[2].value, peak_bytes=v[3].value)

    def sub_csr(self, sub):
        info = self.sub_info(sub)
        rp = np.zeros(info["n"] + 1, dtype=np.int64)
        col = np.zeros(info["nnz"], dtype=np.int64)
        val = np.zeros(info["nnz"], dtype=np.complex128)
        lib().hsref_sub_csr(self.h, int(sub), rp.ctypes.data_as(_c_ll_p), col.ctypes.data_as(_c_ll_p), _p(val))
        return rp, col, val

    def sub_solve(self, sub, rhs):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.zeros_like(rhs)
        _check(lib().hsref_sub_solve(self.h, int(sub), _p(rhs), _p(x)))
        return x

    def global_csr(self):
        nnz = ctypes.c_longlong()
        lib().hsref_global_csr_nnz(self.h, ctypes.byref(nnz))
        rp = np.zeros(self.N + 1, dtype=np.int64)
        col = np.zeros(nnz.value, dtype=np.int64)
        val = np.zeros(nnz.value, dtype=np.complex128)
        lib().hsref_global_csr(self.h, rp.ctypes.data_as(_c_ll_p), col.ctypes.data_as(_c_ll_p), _p(val))
        return rp, col, val

    def gmres(self, b, tol, maxit, rounds=1):
        b = np.ascontiguousarray(b, dtype=np.complex128)
        x = np.zeros(self.N, dtype=np.complex128)
        it, conv, nh = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        hist = np.zeros(maxit + 2)
        fr, tr, sec = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _check(lib().hsref_gmres(self.h, _p(b), _p(x), ctypes.c_double(tol), int(maxit), int(rounds),
                                 ctypes.byref(it), ctypes.byref(conv), _p(hist), ctypes.byref(nh),
                                 ctypes.byref(fr), ctypes.byref(tr), ctypes.byref(sec)))
        return x, dict(iterations=it.value, converged=bool(conv.value), history=hist[: nh.value].tolist(),
                       final_residual=fr.value, true_residual=tr.value, seconds=sec.value)

    def global_direct_solve(self, f):
        f = np.ascontiguousarray(f, dtype=np.complex128)
        u = np.zeros(self.N, dtype=np.complex128)
        _check(lib().hsref_global_direct_solve(self.h, _p(f), _p(u)))
        return u


def blas_active():
    """Whether the shim's large dense products run on OpenBLAS (HSREF_BLAS=0 forces naive loops)."""
    return bool(lib().hsref_blas_active())


def route(dim, rounds, gen_sweep, axis, sign):
    return lib().hsref_route(int(dim), int(rounds), int(gen_sweep), int(axis), int(sign))


def step_of(dim, counts, sweep_index, sub):
    c = (ctypes.c_int * 3)(*counts)
    s = (ctypes.c_int * 3)(*sub)
    return lib().hsref_step_of(int(dim), c, int(sweep_index), s)


class RefFactorization:
    """factorize(const SparseOperator&) on a CSR over a grid range (src/direct.cpp:333-348)."""

    def __init__(self, dim, lo, hi, row_ptr, col, val):
        L = lib()
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int64)
        val = np.ascontiguousarray(val, dtype=np.complex128)
        self.n = len(row_ptr) - 1
        self.h = ctypes.c_void_p()
        fnnz, piv = ctypes.c_longlong(), ctypes.c_longlong(-1)
        rc = L.hsref_factorize(int(dim), (ctypes.c_int * 3)(*lo), (ctypes.c_int * 3)(*hi),
                               ctypes.c_longlong(self.n), row_ptr.ctypes.data_as(_c_ll_p),
                               col.ctypes.data_as(_c_ll_p), _p(val), ctypes.byref(self.h),
                               ctypes.byref(fnnz), ctypes.byref(piv))
        _check(rc, piv.value)
        self.factor_nnz = fnnz.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.hsref_fact_destroy(self.h)
            self.h = None

    def solve(self, rhs):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.zeros_like(rhs)
        _check(lib().hsref_fact_solve(self.h, _p(rhs), _p(x)))
        return x


def pml_operator(dim, n, pad, kappa):
    """tests/test_direct.cpp:14-37 helper, built by the reference."""
    L = lib()
    rows, nnz = ctypes.c_longlong(), ctypes.c_longlong()
    _check(L.hsref_pml_operator(int(dim), int(n), int(pad), ctypes.c_double(kappa), ctypes.byref(rows),
                                ctypes.byref(nnz), None, None, None))
    rp = np.zeros(rows.value + 1, dtype=np.int64)
    col = np.zeros(nnz.value, dtype=np.int64)
    val = np.zeros(nnz.value, dtype=np.complex128)
    _check(L.hsref_pml_operator(int(dim), int(n), int(pad), ctypes.c_double(kappa), ctypes.byref(rows),
                                ctypes.byref(nnz), rp.ctypes.data_as(_c_ll_p), col.ctypes.data_as(_c_ll_p), _p(val)))
    return rp, col, val
