"""Developer check: a larger 3D configuration on the device (timings, memory) with the residual."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_02585_b200 as hs
from paper_2003_02585_b200 import sources
n, parts, pad = int(os.environ.get("N3", "64")), int(os.environ.get("P3", "2")), int(os.environ.get("PAD3", "8"))
kap = 2 * math.pi * float(os.environ.get("F3", "6"))
t = time.perf_counter()
s = hs.DdmSolver(hs.ProblemSetup(3, [n] * 3, [parts] * 3, hs.Medium("constant", kappa=kap), pml_width=pad))
print("device setup+factor s %.2f factor_seconds %.2f" % (time.perf_counter() - t, s.factor_seconds()), flush=True)
f = sources.gaussian_sources(3, s.lo, s.hi, [1.0 / n] * 3, [0.0] * 3, sources.seeded_centers(7, 8, 3), 2.0 / n)
b = s.scale_source(f)
for it in range(2):
    t = time.perf_counter(); reps = []
    U = s.ddm_solve(b, 1, reps, True)
    print("ddm wall s %.3f device sweep s %.4f residual %.3e solves %d" % (time.perf_counter() - t, reps[0].sweep_seconds_total,
          reps[0].round_residuals[0], reps[0].local_solves), flush=True)
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv"], capture_output=True, text=True).stdout)
