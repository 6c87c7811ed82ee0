"""Developer profiling driver (not part of the product): builds a BASELINE configuration's solver
and runs N DDM applications from device-resident b, printing device times. Used under ncu with a
kernel filter to capture one representative solve launch, and with HS_STEP_TIMES for per-macro-step
solve times.

  python tools/profile_cfg.py c3 [--apps N] [--rhs R]
"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2003_02585_b200 as hs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", choices=sorted(bench.CONFIGS))
    ap.add_argument("--apps", type=int, default=2)
    ap.add_argument("--rhs", type=int, default=0)
    a = ap.parse_args()
    bench.select(a.cfg)
    C = bench.CFG
    setup = hs.ProblemSetup(2, [C["n"]] * 2, list(C["parts"]), bench.medium(hs), pml_width=C["pad"])
    t = time.perf_counter()
    s = hs.DdmSolver(setup)
    setup_s = time.perf_counter() - t
    R = a.rhs or C["nrhs"]
    f = bench.make_sources(C["seed"], s.lo, s.hi, [1.0 / C["n"]] * 2, [0.0, 0.0])[:R]
    b = s.scale_source(f)
    db = torch.from_numpy(b.view(np.float64)).cuda()
    du = torch.empty_like(db)
    st = torch.cuda.current_stream().cuda_stream
    out = {"cfg": a.cfg, "rhs": R, "setup_s": setup_s, "factor_s": s.factor_seconds(), "mem": s.memory()}
    for i in range(a.apps):
        reps = s.ddm_solve_device(db.data_ptr(), du.data_ptr(), R, C["rounds"], True, st, want_reports=True)
        mb = s.memory()["max_batch"]  # one report per device batch carries its application's time
        out.setdefault("app_ms", []).append(1e3 * sum(reps[q].sweep_seconds_total for q in range(0, R, mb)))
    out["profile"] = s.profile()
    out["schedule"] = s.schedule_info(C["rounds"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
