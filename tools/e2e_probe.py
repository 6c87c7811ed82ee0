"""Developer probe: where the end-to-end (host buffer) time of one C2 application goes, and
whether per-call times are stable (per-call samples of the host path and the device path)."""
import math, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_02585_b200 as hs
from paper_2003_02585_b200 import sources
s = hs.DdmSolver(hs.ProblemSetup(2, [1024, 1024], [8, 8], hs.Medium("constant", kappa=2 * math.pi * 64), pml_width=32))
f = sources.gaussian_sources(2, s.lo, s.hi, [1.0 / 1024] * 2, [0.0, 0.0], sources.seeded_centers(1000, 16, 2), 2.0 / 1024)
b = s.scale_source(f)
hb = torch.from_numpy(b.view(np.float64)).pin_memory(); hu = torch.empty_like(hb).pin_memory()
db = hb.cuda(); du = torch.empty_like(db)
st = torch.cuda.current_stream().cuda_stream
n = int(os.environ.get("HS_N_CALLS", "20"))
if os.environ.get("HS_SMI"):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                         stdout=subprocess.DEVNULL)
for _ in range(3): s.ddm_solve_device(db.data_ptr(), du.data_ptr(), 16, 1, True, st)
torch.cuda.synchronize()
dev = []
for _ in range(n):
    t = time.perf_counter(); s.ddm_solve_device(db.data_ptr(), du.data_ptr(), 16, 1, True, st); torch.cuda.synchronize()
    dev.append(1e3 * (time.perf_counter() - t))
print("device path per-call ms", [round(x, 1) for x in dev], flush=True)
if os.environ.get("HS_SMI"):
    p.terminate(); p.wait()
for _ in range(3): s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), 16, 1, True)
host = []
for _ in range(n):
    t = time.perf_counter(); s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), 16, 1, True)
    host.append(1e3 * (time.perf_counter() - t))
print("host path per-call ms", [round(x, 1) for x in host], flush=True)
print("equal", bool(torch.equal(du.cpu(), hu)))
