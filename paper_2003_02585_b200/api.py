"""Host-side mirror of the reference's hot-path API over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference (``/root/reference/proj``):

* ``factorize(op) -> Factorization`` with ``solve`` / ``solve_inplace`` / ``stats``
  (include/helmsweep/direct.hpp:22-41);
* ``DdmSolver(setup)`` with ``ddm_solve(b, rounds, report, track_residuals)``,
  ``scale_source``, ``global_op().apply`` (include/helmsweep/sweeper.hpp:70-107), plus a
  batched multi-RHS form (the reference is single-RHS per call);
* ``gmres(...)`` wired as ``run_precond`` wires it (src/harness.cpp:285-305);
* ``ConfigError`` / ``DataError`` / ``SingularMatrixError(pivot_index)``
  (include/helmsweep/common.hpp:18-35).

Every numeric call runs on the GPU through ``libhelmsweep_b200.so``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


class HelmsweepError(RuntimeError):
    pass


class ConfigError(HelmsweepError):
    pass


class DataError(HelmsweepError):
    pass


class SingularMatrixError(HelmsweepError):
    def __init__(self, msg, pivot_index, sub=-1):
        super().__init__(msg)
        self.pivot_index = pivot_index
        self.sub = sub


class CudaError(HelmsweepError):
    pass


def _raise(rc, pivot_index=-1, sub=-1):
    msg = L.last_error()
    if rc == L.HS_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == L.HS_ERR_DATA:
        raise DataError(msg)
    if rc == L.HS_ERR_SINGULAR:
        raise SingularMatrixError(msg, pivot_index, sub)
    if rc == L.HS_ERR_CUDA:
        raise CudaError(msg)
    raise HelmsweepError(msg)


def _dptr(a):
    return a.ctypes.data_as(L.c_dbl_p)


def _as_c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


# ----------------------------------------------------------------------------
# factorization


@dataclass
class SparseOperator:
    """CSR over a grid range (include/helmsweep/operator.hpp:14-25)."""
    dim: int
    lo: Sequence[int]
    hi: Sequence[int]
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def n(self):
        return len(self.row_ptr) - 1


class Factorization:
    def __init__(self, handle, stats):
        self._h = handle
        self._stats = stats

    def __del__(self):
        if getattr(self, "_h", None):
            try:  # at interpreter shutdown the binding may already be torn down
                L.lib().hs_factor_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def stats(self):
        return self._stats

    def solve(self, rhs):
        """Factorization::solve (direct.hpp:28); rhs is (n,) or (R, n) RHS-major."""
        x = np.array(rhs, dtype=np.complex128, copy=True, order="C")
        self.solve_inplace(x)
        return x

    def solve_inplace(self, x):
        if x.dtype != np.complex128 or not x.flags.c_contiguous:
            raise ConfigError("solve_inplace needs a C-contiguous complex128 array")
        n = self._stats.n
        if x.shape[-1] != n:
            raise ConfigError("Factorization::solve: length mismatch")
        nrhs = 1 if x.ndim == 1 else x.shape[0]
        rc = L.lib().hs_factor_solve(self._h, nrhs, _dptr(x))
        if rc:
            _raise(rc)
        return x

    def solve_device(self, ptr, nrhs, stream=0):
        rc = L.lib().hs_factor_solve_device(self._h, nrhs, ctypes.c_void_p(ptr), ctypes.c_void_p(stream))
        if rc:
            _raise(rc)


def factorize(op: SparseOperator, device=0) -> Factorization:
    """factorize(const SparseOperator&) (src/direct.cpp:333-348), on the GPU."""
    lo = (ctypes.c_int * 3)(*(list(op.lo) + [0] * (3 - len(op.lo))))
    hi = (ctypes.c_int * 3)(*(list(op.hi) + [0] * (3 - len(op.hi))))
    rp = np.ascontiguousarray(op.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(op.col, dtype=np.int64)
    val = _as_c128(op.val)
    h = ctypes.c_void_p()
    st = L.FactorStats()
    piv = ctypes.c_int64(-1)
    rc = L.lib().hs_factorize(int(op.dim), lo, hi, ctypes.c_int64(op.n), rp.ctypes.data_as(L.c_i64_p),
                              col.ctypes.data_as(L.c_i64_p), _dptr(val), int(device), ctypes.byref(h),
                              ctypes.byref(st), ctypes.byref(piv))
    if rc:
        _raise(rc, piv.value)
    return Factorization(h, st)


# ----------------------------------------------------------------------------
# DDM solver


@dataclass
class Medium:
    """WaveNumberModel (include/helmsweep/media.hpp:31-55)."""
    kind: str = "constant"
    kappa: float = 0.0
    kappa_down: float = 0.0
    kappa_up: float = 0.0
    axis: int = 1
    eta: float = 0.0
    eps: float = 0.0
    velocity: Optional[np.ndarray] = None  # float32 samples, axis 0 fastest
    vel_n: Sequence[int] = (2, 2, 1)
    vel_origin: Sequence[float] = (0.0, 0.0, 0.0)
    vel_spacing: Sequence[float] = (1.0, 1.0, 0.0)
    omega: float = 0.0


@dataclass
class ProblemSetup:
    """ProblemSetup (include/helmsweep/sweeper.hpp:58-65)."""
    dim: int
    intervals: Sequence[int]
    counts: Sequence[int]
    medium: Medium
    pml_width: int = 30
    pml_strength: float = 2.0
    pml_exponent: int = 2
    interior_lo: Sequence[float] = (0.0, 0.0, 0.0)
    interior_hi: Sequence[float] = (1.0, 1.0, 1.0)
    workers: int = 1

    def to_c(self):
        p = L.Problem()
        d = self.dim
        p.dim = d
        for a in range(3):
            p.interior_lo[a] = self.interior_lo[a] if a < d else 0.0
            p.interior_hi[a] = self.interior_hi[a] if a < d else 1.0
            p.intervals[a] = self.intervals[a] if a < d else 1
            p.counts[a] = self.counts[a] if a < d else 1
        p.pml_width, p.pml_strength, p.pml_exponent = self.pml_width, self.pml_strength, self.pml_exponent
        m = self.medium
        p.medium_kind = {"constant": 0, "two_layered": 1, "gridded": 2}[m.kind]
        p.kappa, p.kappa_down, p.kappa_up = m.kappa, m.kappa_down, m.kappa_up
        p.interface_axis, p.eta, p.eps = m.axis, m.eta, m.eps
        self._vel = None
        if m.kind == "gridded":
            self._vel = np.ascontiguousarray(m.velocity, dtype=np.float32)
            p.vel_dim = d
            for a in range(3):
                p.vel_n[a] = m.vel_n[a] if a < len(m.vel_n) else 1
                p.vel_origin[a] = m.vel_origin[a] if a < len(m.vel_origin) else 0.0
                p.vel_spacing[a] = m.vel_spacing[a] if a < len(m.vel_spacing) else 0.0
            p.vel_c = self._vel.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
            p.omega = m.omega
        p.workers = self.workers
        return p


@dataclass
class SolveReport:
    """SolveReport (include/helmsweep/sweeper.hpp:44-56)."""
    factor_seconds: float = 0.0
    sweep_seconds_total: float = 0.0
    sweep_seconds: List[float] = field(default_factory=list)
    sweep_contrib_norm: List[float] = field(default_factory=list)
    traces_generated: int = 0
    traces_routed: int = 0
    traces_discarded: int = 0
    local_solves: int = 0
    skipped_zero_solves: int = 0
    round_residuals: List[float] = field(default_factory=list)
    median_subdomain_solve_seconds: float = 0.0

    @staticmethod
    def from_c(c: L.SolveReportC):
        return SolveReport(
            c.factor_seconds, c.sweep_seconds_total, list(c.sweep_seconds[: c.n_sweeps]),
            list(c.sweep_contrib_norm[: c.n_sweeps]), c.traces_generated, c.traces_routed, c.traces_discarded,
            c.local_solves, c.skipped_zero_solves, list(c.round_residuals[: c.n_round_residuals]),
            c.median_subdomain_solve_seconds)


@dataclass
class GmresResult:
    """GmresResult (include/helmsweep/krylov.hpp:22-29)."""
    x: np.ndarray
    history: List[float]
    iterations: int
    converged: bool
    final_residual: float
    true_residual: float


class DdmSolver:
    """DdmSolver (src/sweeper.cpp:133-334): factorization at construction, device sweeps."""

    def __init__(self, setup: ProblemSetup, device: int = 0):
        self.setup = setup
        p = setup.to_c()
        h = ctypes.c_void_p()
        sub, piv = ctypes.c_int(-1), ctypes.c_int64(-1)
        rc = self._create(p, int(device), h, sub, piv)
        if rc:
            _raise(rc, piv.value, sub.value)
        self._h = h
        dim, n, ns, fs = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_double()
        lo, hi = (ctypes.c_int * 3)(), (ctypes.c_int * 3)()
        L.lib().hs_ddm_info(h, ctypes.byref(dim), ctypes.byref(n), ctypes.byref(ns), ctypes.byref(fs), lo, hi)
        self.dim, self.global_n, self.nsub = dim.value, n.value, ns.value
        self._factor_seconds = fs.value
        self.lo, self.hi = list(lo), list(hi)

    def _create(self, p, device, h, sub, piv):
        return L.lib().hs_ddm_create(ctypes.byref(p), device, ctypes.byref(h), ctypes.byref(sub), ctypes.byref(piv))

    def __del__(self):
        if getattr(self, "_h", None):
            try:  # at interpreter shutdown the binding may already be torn down
                L.lib().hs_ddm_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def factor_seconds(self):
        return self._factor_seconds

    def sub_stats(self, sub) -> L.FactorStats:
        st = L.FactorStats()
        rc = L.lib().hs_ddm_sub_stats(self._h, int(sub), ctypes.byref(st))
        if rc:
            _raise(rc)
        return st

    def scale_source(self, f):
        f = _as_c128(f)
        b = np.zeros_like(f)
        nrhs = 1 if f.ndim == 1 else f.shape[0]
        if f.shape[-1] != self.global_n:
            raise ConfigError("scale_source: field size mismatch")
        rc = L.lib().hs_ddm_scale_source(self._h, nrhs, _dptr(f), _dptr(b))
        if rc:
            _raise(rc)
        return b

    def ddm_solve(self, b, rounds=1, report: Optional[list] = None, track_residuals=False):
        """One DDM application. b: (N,) or (R, N). Returns u of the same shape; when
        ``report`` is a list it receives one SolveReport per RHS."""
        b = _as_c128(b)
        if b.shape[-1] != self.global_n:
            raise ConfigError("ddm_solve: rhs size mismatch")
        nrhs = 1 if b.ndim == 1 else b.shape[0]
        u = np.zeros_like(b)
        reps = (L.SolveReportC * nrhs)()
        rc = L.lib().hs_ddm_solve(self._h, nrhs, _dptr(b), _dptr(u), int(rounds), int(bool(track_residuals)), reps)
        if rc:
            _raise(rc)
        if report is not None:
            report.extend(SolveReport.from_c(r) for r in reps)
        return u

    def ddm_solve_host_ptr(self, b_ptr, u_ptr, nrhs, rounds=1, track_residuals=False):
        """hs_ddm_solve on raw host pointers (e.g. pinned buffers): H2D, application, D2H."""
        rc = L.lib().hs_ddm_solve(self._h, int(nrhs), ctypes.cast(ctypes.c_void_p(b_ptr), L.c_dbl_p),
                                  ctypes.cast(ctypes.c_void_p(u_ptr), L.c_dbl_p), int(rounds),
                                  int(bool(track_residuals)), None)
        if rc:
            _raise(rc)

    def ddm_solve_device(self, b_ptr, u_ptr, nrhs, rounds=1, track_residuals=False, stream=0, want_reports=False):
        """Device-pointer form (RHS-major complex128); asynchronous on `stream` unless
        reports are requested."""
        reps = (L.SolveReportC * nrhs)() if want_reports else None
        rc = L.lib().hs_ddm_solve_device(self._h, int(nrhs), ctypes.c_void_p(b_ptr), ctypes.c_void_p(u_ptr),
                                         int(rounds), int(bool(track_residuals)), reps, ctypes.c_void_p(stream))
        if rc:
            _raise(rc)
        return [SolveReport.from_c(r) for r in reps] if want_reports else None

    def profile(self):
        """Solve-kernel profile of the last timed batch (hs_ddm_profile)."""
        sec, nb, ns = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        by, fl = ctypes.c_double(), ctypes.c_double()
        rc = L.lib().hs_ddm_profile(self._h, ctypes.byref(sec), ctypes.byref(nb), ctypes.byref(ns),
                                    ctypes.byref(by), ctypes.byref(fl))
        if rc:
            _raise(rc)
        return dict(solve_seconds=sec.value, solve_launches=nb.value, subdomain_solves=ns.value,
                    alg_bytes=by.value, alg_flops=fl.value)

    def apply_op(self, x):
        """global_op().apply(x) (src/operator.cpp:7-17) on the device."""
        x = _as_c128(x)
        y = np.zeros_like(x)
        nrhs = 1 if x.ndim == 1 else x.shape[0]
        rc = L.lib().hs_ddm_apply_op(self._h, nrhs, _dptr(x), _dptr(y))
        if rc:
            _raise(rc)
        return y

    def sub_csr(self, sub):
        """(row_ptr, col, val) of subdomain `sub`'s operator as assembled by the solver (hs_ddm_sub_csr)."""
        n, nnz = ctypes.c_int64(), ctypes.c_int64()
        rc = L.lib().hs_ddm_sub_csr(self._h, int(sub), None, None, None, ctypes.byref(n), ctypes.byref(nnz))
        if rc:
            _raise(rc)
        rp = np.zeros(n.value + 1, dtype=np.int64)
        col = np.zeros(nnz.value, dtype=np.int64)
        val = np.zeros(nnz.value, dtype=np.complex128)
        rc = L.lib().hs_ddm_sub_csr(self._h, int(sub), rp.ctypes.data_as(L.c_i64_p), col.ctypes.data_as(L.c_i64_p),
                                    _dptr(val), None, None)
        if rc:
            _raise(rc)
        return rp, col, val

    def memory(self):
        """Resident factor bytes, solve-state bytes and the device batch width (hs_ddm_memory)."""
        fb, sb, mb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        rc = L.lib().hs_ddm_memory(self._h, ctypes.byref(fb), ctypes.byref(sb), ctypes.byref(mb))
        if rc:
            _raise(rc)
        return {"factor_bytes": fb.value, "state_bytes": sb.value, "max_batch": mb.value}

    def factor_bytes(self):
        return self.memory()["factor_bytes"]

    def batches_per_application(self, nrhs):
        mb = self.memory()["max_batch"]
        return (int(nrhs) + mb - 1) // mb

    def schedule_info(self, rounds=1):
        """Device sweep schedule: macro-steps, widest macro-step, the reference's sequential step
        count and x buffers in flight."""
        v = [ctypes.c_int() for _ in range(4)]
        rc = L.lib().hs_ddm_schedule_info(self._h, int(rounds), *[ctypes.byref(x) for x in v])
        if rc:
            _raise(rc)
        return {"macro_steps": v[0].value, "max_width": v[1].value, "sequential_steps": v[2].value,
                "buffers": v[3].value}

    def global_direct_solve(self, f, stats: Optional[list] = None):
        """global_direct_solve(cfg, f) (src/harness.cpp:185-214): u = A^-1 (J f) on the padded
        global grid with the device sparse-direct factorization of the global operator (built on
        first use, then kept). f: (N,) or (R, N) physical source."""
        f = _as_c128(f)
        u = np.zeros_like(f)
        nrhs = 1 if f.ndim == 1 else f.shape[0]
        st = L.FactorStats()
        rc = L.lib().hs_ddm_global_solve(self._h, nrhs, _dptr(f), _dptr(u), ctypes.byref(st))
        if rc:
            _raise(rc)
        if stats is not None:
            stats.append(st)
        return u

    def gmres(self, b, tol=1e-6, maxit=100, rounds=1, restart=None):
        """gmres(A.apply, ddm_solve, b, cfg) as run_precond wires it (src/harness.cpp:285-305).
        restart=None is the reference's full GMRES; restart=m runs GMRES(m) cycles up to maxit."""
        b = _as_c128(b)
        nrhs = 1 if b.ndim == 1 else b.shape[0]
        x = np.zeros_like(b)
        reps = (L.GmresReportC * nrhs)()
        if restart is None:
            rc = L.lib().hs_gmres(self._h, nrhs, _dptr(b), _dptr(x), float(tol), int(maxit), int(rounds), reps)
        else:
            rc = L.lib().hs_gmres_restarted(self._h, nrhs, _dptr(b), _dptr(x), float(tol), int(maxit), int(restart),
                                            int(rounds), reps)
        if rc:
            _raise(rc)
        out = []
        for r in range(nrhs):
            c = reps[r]
            out.append(GmresResult(x if b.ndim == 1 else x[r], list(c.history[: c.n_history]), c.iterations,
                                   bool(c.converged), c.final_residual, c.true_residual))
        return out[0] if b.ndim == 1 else out


def gmres(op, pc, b, tol=1e-6, maxit=100, restart=None, device=0):
    """gmres(op, pc, b, cfg) (include/helmsweep/krylov.hpp:30-36) for any LinearMaps: `op` and
    `pc` (None = identity) map an (R, n) complex128 array to an (R, n) array, like
    a LinearMap (krylov.hpp:30) applied to R CVectors. The Krylov vectors and reductions live on the device
    (hs_gmres_general); the callbacks run on the host. b: (n,) or (R, n)."""
    b = _as_c128(b)
    single = b.ndim == 1
    B = b.reshape(1, -1) if single else b
    nrhs, n = B.shape
    x = np.zeros_like(B)
    reps = (L.GmresReportC * nrhs)()
    err = []

    def wrap(f):
        def cb(_user, r, px, py, _stream):
            try:
                xin = np.ctypeslib.as_array(ctypes.cast(px, ctypes.POINTER(ctypes.c_double)), shape=(r, 2 * n))
                yout = np.ctypeslib.as_array(ctypes.cast(py, ctypes.POINTER(ctypes.c_double)), shape=(r, 2 * n))
                y = np.ascontiguousarray(f(xin.view(np.complex128).copy()), dtype=np.complex128).reshape(r, n)
                yout[:] = y.view(np.float64)
                return 0
            except Exception as e:  # reported to the caller after the C call returns
                err.append(e)
                return 1
        return L.LINOP_FN(cb)

    c_op = wrap(op)
    c_pc = wrap(pc) if pc is not None else ctypes.cast(None, L.LINOP_FN)
    rc = L.lib().hs_gmres_general(int(device), n, nrhs, c_op, c_pc, None, 0, _dptr(B), _dptr(x), float(tol), int(maxit),
                                  int(maxit if restart is None else restart), reps)
    if err:
        raise err[0]
    if rc:
        _raise(rc)
    out = []
    for r in range(nrhs):
        c = reps[r]
        out.append(GmresResult(x[r], list(c.history[: c.n_history]), c.iterations, bool(c.converged), c.final_residual,
                               c.true_residual))
    return out[0] if single else out


def route_trace(dim, rounds, gen_sweep, axis, sign):
    """route_trace (src/sweeper.cpp:58-73) as implemented by the product's host layer."""
    return int(L.lib().hs_route_trace(dim, rounds, gen_sweep, axis, sign))


def kernel_launches():
    return int(L.lib().hs_kernel_launches())


def device_count():
    return int(L.lib().hs_device_count())


# ---------------------------------------------------------------------------------------------
# On-disk formats (byte-exact with the reference): HSVG velocity grids, HSFD field dumps.

@dataclass
class VelocityGrid:
    """VelocityGrid (include/helmsweep/media.hpp:11-20): samples c (float32, axis 0 fastest)."""
    dim: int
    n: Sequence[int]
    origin: Sequence[float]
    spacing: Sequence[float]
    c: np.ndarray

    def medium(self, omega: float) -> Medium:
        """The gridded WaveNumberModel kappa = omega / c(x) (include/helmsweep/media.hpp:31-55)."""
        return Medium("gridded", velocity=self.c, vel_n=tuple(self.n), vel_origin=tuple(self.origin),
                      vel_spacing=tuple(self.spacing), omega=omega)


@dataclass
class FieldDump:
    """FieldDump (include/helmsweep/harness.hpp:12-15): a complex field on a grid range."""
    dim: int
    lo: Sequence[int]
    hi: Sequence[int]
    h: Sequence[float]
    origin: Sequence[float]
    values: np.ndarray


def _read_vel(fn, path):
    dim, n = ctypes.c_int(), (ctypes.c_int * 3)()
    org, sp, count = (ctypes.c_double * 3)(), (ctypes.c_double * 3)(), ctypes.c_int64()
    rc = fn(str(path).encode(), ctypes.byref(dim), n, org, sp, None, 0, ctypes.byref(count))
    if rc:
        _raise(rc)
    c = np.empty(count.value, dtype=np.float32)
    rc = fn(str(path).encode(), ctypes.byref(dim), n, org, sp, c.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
            count.value, ctypes.byref(count))
    if rc:
        _raise(rc)
    return VelocityGrid(dim.value, list(n), list(org), list(sp), c)


def read_velocity_grid(path) -> VelocityGrid:
    """read_velocity_grid (src/media.cpp:58-84): the HSVG binary layout."""
    return _read_vel(L.lib().hs_read_velocity_grid, path)


def read_velocity_csv(path) -> VelocityGrid:
    """read_velocity_csv (src/media.cpp:102-130): header "dim,n..,origin..,spacing..", one value per line."""
    return _read_vel(L.lib().hs_read_velocity_csv, path)


def write_velocity_grid(path, g: VelocityGrid) -> None:
    """write_velocity_grid (src/media.cpp:86-100)."""
    c = np.ascontiguousarray(g.c, dtype=np.float32)
    n = (ctypes.c_int * 3)(*(list(g.n) + [1] * 3)[:3])
    rc = L.lib().hs_write_velocity_grid(str(path).encode(), int(g.dim), n, (ctypes.c_double * 3)(*g.origin[:3]),
                                        (ctypes.c_double * 3)(*g.spacing[:3]),
                                        c.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    if rc:
        _raise(rc)


def write_field(path, dim, lo, hi, h, origin, u) -> None:
    """write_field (src/harness.cpp:32-53): u over the grid range [lo, hi] (axis 0 fastest)."""
    u = _as_c128(u).ravel()
    lo3, hi3 = (list(lo) + [0] * 3)[:3], (list(hi) + [0] * 3)[:3]
    count = int(np.prod([hi3[a] - lo3[a] + 1 for a in range(dim)]))
    if u.size != count:
        raise ConfigError("write_field: size mismatch")
    rc = L.lib().hs_write_field(str(path).encode(), int(dim), (ctypes.c_int * 3)(*lo3), (ctypes.c_int * 3)(*hi3),
                                (ctypes.c_double * 3)(*(list(h) + [0.0] * 3)[:3]),
                                (ctypes.c_double * 3)(*(list(origin) + [0.0] * 3)[:3]), _dptr(u))
    if rc:
        _raise(rc)


def read_field(path) -> FieldDump:
    """read_field (src/harness.cpp:55-83)."""
    dim, lo, hi = ctypes.c_int(), (ctypes.c_int * 3)(), (ctypes.c_int * 3)()
    h, org, count = (ctypes.c_double * 3)(), (ctypes.c_double * 3)(), ctypes.c_int64()
    fn = L.lib().hs_read_field
    rc = fn(str(path).encode(), ctypes.byref(dim), lo, hi, h, org, None, 0, ctypes.byref(count))
    if rc:
        _raise(rc)
    u = np.empty(count.value, dtype=np.complex128)
    rc = fn(str(path).encode(), ctypes.byref(dim), lo, hi, h, org, _dptr(u), count.value, ctypes.byref(count))
    if rc:
        _raise(rc)
    return FieldDump(dim.value, list(lo), list(hi), list(h), list(org), u)


# ---------------------------------------------------------------------------------------------
# Pipeline cost model (include/helmsweep/pipeline.hpp, src/pipeline.cpp:20-111)

@dataclass
class PipelineCost:
    average_per_rhs: float
    idle_fraction: float


@dataclass
class PipelineSimulation:
    completion_times: np.ndarray
    makespan: float
    average_per_rhs: float


def _counts3(counts):
    return (ctypes.c_int * 3)(*(list(counts) + [1, 1, 1])[:3])


def average_time_per_rhs(dim, counts, n_rhs, n_iter, t0) -> PipelineCost:
    """Closed form 2^dim n_iter t0 + steps / n_rhs t0 (src/pipeline.cpp:20-27)."""
    avg, idle = ctypes.c_double(), ctypes.c_double()
    rc = L.lib().hs_pipeline_cost(int(dim), _counts3(counts), int(n_rhs), int(n_iter), float(t0),
                                  ctypes.byref(avg), ctypes.byref(idle))
    if rc:
        _raise(rc)
    return PipelineCost(avg.value, idle.value)


def simulate_pipeline(dim, counts, n_rhs, n_iter, t0) -> PipelineSimulation:
    """Discrete-event schedule of (rhs, sweep, subdomain) tasks (src/pipeline.cpp:29-111)."""
    comp = np.zeros(int(n_rhs), dtype=np.float64)
    mk, avg = ctypes.c_double(), ctypes.c_double()
    rc = L.lib().hs_pipeline_simulate(int(dim), _counts3(counts), int(n_rhs), int(n_iter), float(t0), _dptr(comp),
                                      ctypes.byref(mk), ctypes.byref(avg))
    if rc:
        _raise(rc)
    return PipelineSimulation(comp, mk.value, avg.value)
