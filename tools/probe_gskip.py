"""Developer probe: C3 with only the first NZ right-hand sides nonzero (the others exactly zero):
device ms per 64-RHS application, with and without HS_NO_GROUP_SKIP (run twice)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
import paper_2003_02585_b200 as hs

bench.select("c3")
C = bench.CFG
setup = hs.ProblemSetup(2, [C["n"]] * 2, list(C["parts"]), bench.medium(hs), pml_width=C["pad"])
s = hs.DdmSolver(setup)
R = C["nrhs"]
f = bench.make_sources(C["seed"], s.lo, s.hi, [1.0 / C["n"]] * 2, [0.0, 0.0])[:R]
b = s.scale_source(f)
nzr = int(os.environ.get("NZ", "8"))
b[nzr:] = 0
db = torch.from_numpy(b.view(np.float64)).cuda()
du = torch.empty_like(db)
st = torch.cuda.current_stream().cuda_stream
ms = []
for i in range(4):
    reps = s.ddm_solve_device(db.data_ptr(), du.data_ptr(), R, C["rounds"], True, st, want_reports=True)
    ms.append(round(1e3 * reps[0].sweep_seconds_total, 2))
print("NZ", nzr, "skip_off", os.environ.get("HS_NO_GROUP_SKIP"), "app_ms", ms, "solve_s", round(s.profile()["solve_seconds"], 4))
