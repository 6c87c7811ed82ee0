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
