"""Developer check: a moderate 3D configuration through the device path against the numpy oracle."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_02585_b200 as hs
from oracle import hs_oracle as O
n, parts, pad = int(os.environ.get("N3", "32")), int(os.environ.get("P3", "2")), int(os.environ.get("PAD3", "6"))
kap = 2 * math.pi * float(os.environ.get("F3", "3"))
t = time.perf_counter()
s = hs.DdmSolver(hs.ProblemSetup(3, [n] * 3, [parts] * 3, hs.Medium("constant", kappa=kap), pml_width=pad))
print("device setup+factor s", time.perf_counter() - t, "factor_seconds", s.factor_seconds())
so = O.DdmSolver(O.ProblemSetup(O.Box(3), [n, n, n], [parts] * 3, O.Medium("constant", kappa=kap), O.PmlSpec(width=pad)))
f = O.gaussian_source(so.ggrid, O.Box(3), [[0.5, 0.5, 0.5], [0.3, 0.6, 0.45]], 2.0 / n)
b = so.scale_source(f).T.copy()
t = time.perf_counter(); reps = []
U = s.ddm_solve(b, 1, reps, True)
print("device ddm s", time.perf_counter() - t, "sweep device s", reps[0].sweep_seconds_total)
for r in range(2):
    t = time.perf_counter()
    uo, ro = so.ddm_solve(b[r].copy(), 1, True)
    print("oracle s", time.perf_counter() - t, "rel", np.linalg.norm(U[r] - uo) / np.linalg.norm(uo),
          "counters", [reps[r].local_solves, reps[r].skipped_zero_solves], [ro.local_solves, ro.skipped_zero_solves])
