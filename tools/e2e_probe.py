"""Developer probe: where the end-to-end (host buffer) time of one C2 application goes."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_02585_b200 as hs
from paper_2003_02585_b200 import sources
s = hs.DdmSolver(hs.ProblemSetup(2, [1024, 1024], [8, 8], hs.Medium("constant", kappa=2 * math.pi * 64), pml_width=32))
f = sources.gaussian_sources(2, s.lo, s.hi, [1.0 / 1024] * 2, [0.0, 0.0], sources.seeded_centers(1000, 16, 2), 2.0 / 1024)
b = s.scale_source(f)
hb = torch.from_numpy(b.view(np.float64)).pin_memory(); hu = torch.empty_like(hb).pin_memory()
db = hb.cuda(); du = torch.empty_like(db)
for _ in range(3): s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), 16, 1, True)
torch.cuda.synchronize()
t = time.perf_counter(); n = 5
for _ in range(n): s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), 16, 1, True)
print("e2e host-ptr ms", 1e3 * (time.perf_counter() - t) / n)
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): s.ddm_solve_device(db.data_ptr(), du.data_ptr(), 16, 1, True, st)
e1.record(); torch.cuda.synchronize(); print("device ms", e0.elapsed_time(e1) / n)
e0.record()
for _ in range(n): db.copy_(hb, non_blocking=True)
e1.record(); torch.cuda.synchronize(); print("H2D ms", e0.elapsed_time(e1) / n, "GB/s", hb.numel() * 8 / (e0.elapsed_time(e1) / n) / 1e6)
e0.record()
for _ in range(n): hu.copy_(du, non_blocking=True)
e1.record(); torch.cuda.synchronize(); print("D2H ms", e0.elapsed_time(e1) / n)
