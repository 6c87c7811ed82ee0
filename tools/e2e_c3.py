"""Developer probe: the C3 host-buffer path (hs_ddm_solve with pinned buffers): per-call ms, and with
HS_STREAM_TRACE=path the timeline of one streamed batch (tile copies in, macro-steps, u tiles out)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
import paper_2003_02585_b200 as hs

bench.select("c3")
C = bench.CFG
setup = hs.ProblemSetup(2, [C["n"]] * 2, list(C["parts"]), bench.medium(hs), pml_width=C["pad"])
s = hs.DdmSolver(setup)
R = int(os.environ.get("R", C["nrhs"]))
f = bench.make_sources(C["seed"], s.lo, s.hi, [1.0 / C["n"]] * 2, [0.0, 0.0])[:R]
b = s.scale_source(f)
hb = torch.from_numpy(b.view(np.float64)).pin_memory(); hu = torch.empty_like(hb).pin_memory()
tr = os.environ.pop("HS_STREAM_TRACE", None)
for _ in range(2): s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), R, C["rounds"], True)
ts = []
for _ in range(4):
    t = time.perf_counter(); s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), R, C["rounds"], True); ts.append(1e3 * (time.perf_counter() - t))
print("host path per-call ms", [round(x, 1) for x in ts], "bytes each way", hb.numel() * 8)
if tr:
    os.environ["HS_STREAM_TRACE"] = tr
    s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), min(R, 32), C["rounds"], True)
    import pandas as pd
    d = pd.read_csv(tr)
    for w in ("h2d_done", "mstep_solve_start", "u_final", "d2h_done", "compute_end"):
        e = d[d.what == w]
        print(f"{w:18s} n={len(e):4d} first {e.ms.min():8.2f} last {e.ms.max():8.2f}")
