"""Profiling driver: C2 workload, a few DDM applications (for ncu / nsight captures)."""
import math, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_02585_b200 as hs
from paper_2003_02585_b200 import sources
n = int(os.environ.get("HS_N", "1024")); parts = int(os.environ.get("HS_P", "8")); pad = int(os.environ.get("HS_PAD", "32"))
kap = 2 * math.pi * float(os.environ.get("HS_F", "64")); R = int(os.environ.get("HS_R", "16")); reps = int(os.environ.get("HS_REPS", "3"))
s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [parts, parts], hs.Medium("constant", kappa=kap), pml_width=pad))
f = sources.gaussian_sources(2, s.lo, s.hi, [1.0 / n] * 2, [0.0, 0.0], sources.seeded_centers(1000, R, 2), 2.0 / n)
b = s.scale_source(f)
for i in range(reps):
    t = time.perf_counter(); rep = []; u = s.ddm_solve(b, 1, rep, True)
    print(f"app {i}: {1e3*(time.perf_counter()-t):.1f} ms wall, device {1e3*rep[0].sweep_seconds_total:.1f} ms", s.profile() if i == reps - 1 else "")
print("factor_seconds", s.factor_seconds())
