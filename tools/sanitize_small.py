"""Developer check: a small wide-batch DDM application (20 RHS, 2 rounds) and a factor solve, meant to
run under compute-sanitizer (memcheck) -- exercises the block loops at 16- and 8-RHS widths, the
staged finalize and the fused accumulate on a problem small enough for the tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_02585_b200 as hs
import math
s = hs.DdmSolver(hs.ProblemSetup(2, [72, 72], [3, 2], hs.Medium("constant", kappa=2 * math.pi * 6), pml_width=8))
g = np.random.default_rng(3)
b = g.standard_normal((20, s.global_n)) + 1j * g.standard_normal((20, s.global_n))
u = s.ddm_solve(b, 2, None, True)
u1 = s.ddm_solve(b[:3], 2, None, True)
print("finite", bool(np.isfinite(u).all()), "batch-independent", float(np.abs(u[:3] - u1).max() / np.abs(u1).max()))
# sparse sources (zero-group skip, half-group narrowing, column order): 41 columns, some all zero
n = [64, 64]
s2 = hs.DdmSolver(hs.ProblemSetup(2, n, [4, 4], hs.Medium("constant", kappa=2 * math.pi * 4), pml_width=6))
gx = s2.hi[0] - s2.lo[0] + 1
B = np.zeros((41, s2.global_n), complex)
for c in range(41):
    if c % 7 == 3:
        continue
    ix, iy = g.integers(2, n[0] - 2), g.integers(2, n[1] - 2)
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            B[c, (ix + dx - s2.lo[0]) + gx * (iy + dy - s2.lo[1])] = g.standard_normal() + 1j * g.standard_normal()
reps = []
U = s2.ddm_solve(B, 2, reps, True)
u5 = s2.ddm_solve(B[5], 2, None, True)
print("sparse finite", bool(np.isfinite(U).all()), "column 5 vs single", float(np.abs(U[5] - u5).max() / np.abs(u5).max()),
      "zero column stays zero", not np.any(U[3]))
