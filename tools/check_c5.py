"""Developer run of BASELINE config 5 (3D, 128^3 + 12-cell PML, 4x4x4 subdomains of 57^3 nodes,
omega = 2 pi 12, 8 seeded sources): device factorization and one DDM application (8 sweeps)."""
import json, math, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_02585_b200 as hs
from paper_2003_02585_b200 import sources
n, parts, pad, kap, R = 128, 4, 12, 2 * math.pi * 12, 8
out = {"config": "C5: 3D constant medium, 128^3 + 12-cell PML, 4x4x4 subdomains, omega = 2 pi 12, 8 RHS"}
t = time.perf_counter()
s = hs.DdmSolver(hs.ProblemSetup(3, [n] * 3, [parts] * 3, hs.Medium("constant", kappa=kap), pml_width=pad))
out["setup_seconds"] = time.perf_counter() - t
out["factor_seconds"] = s.factor_seconds()
st = s.sub_stats(21)
out["interior_sub_factor_nnz"] = st.factor_nnz
print(json.dumps(out), flush=True)
f = sources.gaussian_sources(3, s.lo, s.hi, [1.0 / n] * 3, [0.0] * 3, sources.seeded_centers(1000, R, 3), 2.0 / n)
b = s.scale_source(f)
for it in range(2):
    t = time.perf_counter(); reps = []
    U = s.ddm_solve(b, 1, reps, True)
    out[f"ddm_wall_s_{it}"] = time.perf_counter() - t
    out["sweep_device_s"] = reps[0].sweep_seconds_total
    out["round_residual"] = [r.round_residuals[0] for r in reps]
    out["local_solves"] = reps[0].local_solves
    out["skipped"] = reps[0].skipped_zero_solves
out["rhs_per_s_device"] = R / out["sweep_device_s"]
# the solve launches of the last application: algorithmic bytes (packed factor entries the passes
# multiply + the vectors) over their CUDA-event time; at 8 RHS the solve is HBM-bound (4 flop / B)
pr = s.profile()
hbm = 6551.0
try:
    hbm = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass
out["solve"] = {"seconds": pr["solve_seconds"], "launches": pr["solve_launches"], "alg_bytes": pr["alg_bytes"],
                "alg_flops": pr["alg_flops"], "achieved_gbs": pr["alg_bytes"] / pr["solve_seconds"] / 1e9,
                "hbm_peak_gbs": hbm, "hbm_frac": pr["alg_bytes"] / pr["solve_seconds"] / 1e9 / hbm,
                "tflops": pr["alg_flops"] / pr["solve_seconds"] / 1e12}
out["gpu_mem_used"] = subprocess.run(["nvidia-smi", "--query-gpu=memory.used,memory.total", "--format=csv,noheader"],
                                     capture_output=True, text=True).stdout.strip()
print(json.dumps(out), flush=True)
json.dump(out, open("gpurun_out/c5.json", "w"), indent=1)
