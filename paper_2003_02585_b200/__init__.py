"""helmsweep on B200: the trace-transfer diagonal-sweeping DDM hot path of arXiv 2003.02585
as hand-written sm_100a CUDA behind a C-ABI (include/helmsweep_b200.h).

Python here is only the test/bench plumbing over the C-ABI; see ``api`` for the mirror of
the reference's Factorization / DdmSolver / gmres interface and its on-disk formats.
"""
from .api import (ConfigError, CudaError, DataError, DdmSolver, Factorization, FieldDump, GmresResult,
                  HelmsweepError, Medium, ProblemSetup, SingularMatrixError, SolveReport, SparseOperator,
                  VelocityGrid, average_time_per_rhs, device_count, factorize, gmres, kernel_launches, read_field, read_velocity_csv,
                  read_velocity_grid, route_trace, simulate_pipeline, write_field, write_velocity_grid)
from ._lib import LIB_PATH

__all__ = ["ConfigError", "CudaError", "DataError", "DdmSolver", "Factorization", "FieldDump", "GmresResult",
           "HelmsweepError", "Medium", "ProblemSetup", "SingularMatrixError", "SolveReport", "SparseOperator",
           "VelocityGrid", "average_time_per_rhs", "device_count", "factorize", "gmres", "kernel_launches", "read_field", "read_velocity_csv",
           "read_velocity_grid", "route_trace", "simulate_pipeline", "write_field", "write_velocity_grid", "LIB_PATH"]
