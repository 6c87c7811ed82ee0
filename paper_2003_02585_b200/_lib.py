"""ctypes binding of ``libhelmsweep_b200.so`` (C-ABI: include/helmsweep_b200.h).

The library is built in-tree by ``paper_2003_02585_b200/build.py`` (or
``__graft_entry__.build()``). Loading fails loudly when it is missing: there is no CPU
fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HS_LIB_PATH") or os.path.join(HERE, "libhelmsweep_b200.so")  # override: dev variants

HS_OK, HS_ERR_CONFIG, HS_ERR_DATA, HS_ERR_SINGULAR, HS_ERR_CUDA, HS_ERR_INTERNAL = range(6)
HS_MAX_SWEEPS = 64
HS_MAX_ROUNDS = 16
HS_MAX_GMRES_HISTORY = 257

c_int_p = ctypes.POINTER(ctypes.c_int)
c_i64_p = ctypes.POINTER(ctypes.c_int64)
c_dbl_p = ctypes.POINTER(ctypes.c_double)


class FactorStats(ctypes.Structure):
    """FactorStats (include/helmsweep/direct.hpp:10-17)."""
    _fields_ = [("n", ctypes.c_int64), ("matrix_nnz", ctypes.c_int64), ("factor_nnz", ctypes.c_int64),
                ("peak_bytes", ctypes.c_int64), ("factor_seconds", ctypes.c_double)]

    def fill_ratio(self):
        return self.factor_nnz / self.matrix_nnz if self.matrix_nnz else 0.0


class Problem(ctypes.Structure):
    """ProblemSetup (include/helmsweep/sweeper.hpp:58-65)."""
    _fields_ = [
        ("dim", ctypes.c_int),
        ("interior_lo", ctypes.c_double * 3), ("interior_hi", ctypes.c_double * 3),
        ("intervals", ctypes.c_int * 3), ("counts", ctypes.c_int * 3),
        ("pml_width", ctypes.c_int), ("pml_strength", ctypes.c_double), ("pml_exponent", ctypes.c_int),
        ("medium_kind", ctypes.c_int), ("kappa", ctypes.c_double),
        ("kappa_down", ctypes.c_double), ("kappa_up", ctypes.c_double),
        ("interface_axis", ctypes.c_int), ("eta", ctypes.c_double), ("eps", ctypes.c_double),
        ("vel_dim", ctypes.c_int), ("vel_n", ctypes.c_int * 3),
        ("vel_origin", ctypes.c_double * 3), ("vel_spacing", ctypes.c_double * 3),
        ("vel_c", ctypes.POINTER(ctypes.c_float)), ("omega", ctypes.c_double),
        ("workers", ctypes.c_int),
    ]


class SolveReportC(ctypes.Structure):
    """SolveReport (include/helmsweep/sweeper.hpp:44-56)."""
    _fields_ = [
        ("factor_seconds", ctypes.c_double), ("sweep_seconds_total", ctypes.c_double),
        ("median_subdomain_solve_seconds", ctypes.c_double),
        ("traces_generated", ctypes.c_int64), ("traces_routed", ctypes.c_int64),
        ("traces_discarded", ctypes.c_int64), ("local_solves", ctypes.c_int64),
        ("skipped_zero_solves", ctypes.c_int64),
        ("n_sweeps", ctypes.c_int), ("n_round_residuals", ctypes.c_int),
        ("sweep_seconds", ctypes.c_double * HS_MAX_SWEEPS),
        ("sweep_contrib_norm", ctypes.c_double * HS_MAX_SWEEPS),
        ("round_residuals", ctypes.c_double * HS_MAX_ROUNDS),
    ]


class GmresReportC(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("final_residual", ctypes.c_double), ("true_residual", ctypes.c_double),
                ("n_history", ctypes.c_int), ("history", ctypes.c_double * HS_MAX_GMRES_HISTORY)]


# Callbacks of the partitioned solver (hs_exchange_fn / hs_allreduce_fn)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, c_int_p, c_i64_p, c_i64_p, c_i64_p,
                               c_i64_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
# hs_linop_fn: y = Op x on nrhs RHS-major vectors (host or device pointers), optional stream
LINOP_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

# Every symbol declared in include/helmsweep_b200.h, with its ctypes signature.
SIGNATURES = {
    "hs_last_error": (ctypes.c_char_p, []),
    "hs_device_count": (ctypes.c_int, []),
    "hs_kernel_launches": (ctypes.c_int64, []),
    "hs_factorize": (ctypes.c_int, [ctypes.c_int, c_int_p, c_int_p, ctypes.c_int64, c_i64_p, c_i64_p, c_dbl_p,
                                    ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(FactorStats),
                                    c_i64_p]),
    "hs_factor_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dbl_p]),
    "hs_factor_solve_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "hs_factor_stats_get": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(FactorStats)]),
    "hs_factor_destroy": (None, [ctypes.c_void_p]),
    "hs_ddm_create": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                     c_int_p, c_i64_p]),
    "hs_ddm_destroy": (None, [ctypes.c_void_p]),
    "hs_ddm_info": (ctypes.c_int, [ctypes.c_void_p, c_int_p, c_i64_p, c_int_p, c_dbl_p, c_int_p, c_int_p]),
    "hs_ddm_sub_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(FactorStats)]),
    "hs_ddm_scale_source": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dbl_p, c_dbl_p]),
    "hs_ddm_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dbl_p, c_dbl_p, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(SolveReportC)]),
    "hs_ddm_solve_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int, ctypes.c_int, ctypes.POINTER(SolveReportC),
                                           ctypes.c_void_p]),
    "hs_ddm_apply_op": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dbl_p, c_dbl_p]),
    "hs_ddm_global_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dbl_p, c_dbl_p,
                                           ctypes.POINTER(FactorStats)]),
    "hs_ddm_schedule_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int)]),
    "hs_pipeline_cost": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, c_dbl_p, c_dbl_p]),
    "hs_pipeline_simulate": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                            ctypes.c_double, c_dbl_p, c_dbl_p, c_dbl_p]),
    "hs_read_velocity_grid": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                             c_dbl_p, c_dbl_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int64,
                                             ctypes.POINTER(ctypes.c_int64)]),
    "hs_write_velocity_grid": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), c_dbl_p,
                                              c_dbl_p, ctypes.POINTER(ctypes.c_float)]),
    "hs_read_velocity_csv": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                            c_dbl_p, c_dbl_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int64,
                                            ctypes.POINTER(ctypes.c_int64)]),
    "hs_write_field": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int), c_dbl_p, c_dbl_p, c_dbl_p]),
    "hs_read_field": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int), c_dbl_p, c_dbl_p, c_dbl_p, ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64)]),
    "hs_gmres": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dbl_p, c_dbl_p, ctypes.c_double, ctypes.c_int,
                                ctypes.c_int, ctypes.POINTER(GmresReportC)]),
    "hs_gmres_restarted": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dbl_p, c_dbl_p, ctypes.c_double,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(GmresReportC)]),
    "hs_gmres_general": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int, LINOP_FN, LINOP_FN, ctypes.c_void_p,
                                        ctypes.c_int, c_dbl_p, c_dbl_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(GmresReportC)]),
    "hs_ddm_profile": (ctypes.c_int, [ctypes.c_void_p, c_dbl_p, c_i64_p, c_i64_p, c_dbl_p, c_dbl_p]),
    "hs_route_trace": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "hs_partition_owners": (ctypes.c_int, [ctypes.c_int, c_int_p, ctypes.c_int, c_int_p]),
    "hs_partition_traffic": (ctypes.c_int, [ctypes.c_int, c_int_p, ctypes.c_int, ctypes.c_int, c_int_p, c_int_p,
                                            c_i64_p, c_i64_p, c_i64_p]),
    "hs_ddm_create_partitioned": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                 c_int_p, EXCHANGE_FN, ALLREDUCE_FN, ctypes.c_void_p,
                                                 ctypes.POINTER(ctypes.c_void_p), c_int_p, c_i64_p]),
    "hs_nccl_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ubyte)]),
    "hs_nccl_version": (ctypes.c_int, [c_int_p]),
    "hs_ddm_create_nccl": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.c_int, ctypes.c_int, ctypes.c_int, c_int_p,
                                          ctypes.POINTER(ctypes.c_ubyte), ctypes.POINTER(ctypes.c_void_p), c_int_p,
                                          c_i64_p]),
    "hs_ddm_sub_csr": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_i64_p, c_i64_p, c_dbl_p, c_i64_p, c_i64_p]),
    "hs_ddm_memory": (ctypes.c_int, [ctypes.c_void_p, c_i64_p, c_i64_p, c_int_p]),
    "hs_ddm_partition_info": (ctypes.c_int, [ctypes.c_void_p, c_int_p, c_int_p, c_int_p, c_i64_p, c_i64_p]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"helmsweep_b200 CUDA library missing: {LIB_PATH}. Build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback).")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error():
    return lib().hs_last_error().decode()
