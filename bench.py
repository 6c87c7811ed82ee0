"""Benchmark: RHS/s through full 2^n diagonal sweeps (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1], "C2"): 2D constant medium, 1024^2 interior + 32-cell PML,
omega = 2 pi 64 (c = 1), 8x8 checkerboard subdomains each with its own 32-cell PML, 16 RHS =
Gaussian point sources (sigma = 2h, unit amplitude) at seeded uniform interior locations,
complex128, direct-solver mode: one DDM application = 1 round of 4 diagonal sweeps with the
per-round residual the reference's run_direct tracks (src/harness.cpp:269-283).

A step is one DDM application over the batch of 16 RHS (lockstep-batched through every
subdomain solve). ``value`` = RHS/s with b already resident in HBM, device-timed with CUDA
events; ``e2e`` = the same through hs_ddm_solve with pinned host buffers (H2D of b and D2H of
u inside the timed region). Multi-GPU (torchrun): one process per GPU, each rank sweeps its own
16-RHS batch against its own resident factors (RHS are independent units; no data-path
collective) -> weak scaling, time = max over ranks.

``--impl reference`` runs the reference's own CPU implementation (oracle/_ref, the unmodified
reference compiled in place) on the host cores, one RHS per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RHS/sec through full 2^n diagonal sweeps"
WORKLOAD = ("C2: 2D constant medium c=1, 1024^2 grid + 32-cell PML, omega=2pi*64, 8x8 subdomains, "
            "16 RHS seeded Gaussian sources (sigma=2h), direct-solver mode (1 round = 4 diagonal sweeps, "
            "per-round residual)")
CFG = dict(dim=2, n=1024, parts=(8, 8), pad=32, kappa=2 * math.pi * 64, nrhs=16, rounds=1)


def ref_config():
    return {"dim": 2, "grid.n": [CFG["n"]] * 2, "partition": list(CFG["parts"]), "pml.width": CFG["pad"],
            "media.kind": "constant", "media.kappa": CFG["kappa"]}


def make_sources(seed, lo, hi, hgrid, origin):
    from paper_2003_02585_b200 import sources
    cen = sources.seeded_centers(seed, CFG["nrhs"], 2)
    return sources.gaussian_sources(2, lo, hi, hgrid, origin, cen, 2.0 / CFG["n"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for nme, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(nme)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    """HBM copy bandwidth from MEASURED_PEAKS.json (driver-written) and the FP64 tensor-core
    (DMMA) peak measured by tools/bench_fp64.cu (profiles/fp64_peak.json)."""
    hbm, kind = 6650.0, "fallback"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm, kind = float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        pass
    fp64 = 37.1
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            fp64 = float(json.load(f)["dmma_tflops"])
    except Exception:
        pass
    return hbm, kind, fp64


def ncu_traffic():
    """Per-launch DRAM traffic of the solve kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "solve_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_baseline_sample(b0, u0=None):
    """oracle/_ref (the reference compiled in place) on this host's cores: DdmSolver factorizes
    all 64 subdomains, then one RHS of the workload through one DDM application. With u0 (the
    device result for the same RHS) it also reports the relative L2 difference -- parity at the
    bench's own configuration (north_star: <= 1e-9)."""
    try:
        from oracle import ref
        if not ref.available():
            return {"value": None, "unit": "RHS/s", "cores": 0, "kind": "reference",
                    "sample": "unavailable: oracle/_ref not built"}
        cores = os.cpu_count() or 1
        s = ref.RefSolver(ref_config(), cores)
        t0 = time.perf_counter()
        u, rep = s.ddm_solve(b0, CFG["rounds"], True)
        dt = time.perf_counter() - t0
        out = {"value": 1.0 / dt, "unit": "RHS/s", "cores": cores, "kind": "reference",
               "sample": f"1 of the 16 RHS through one full DDM application (4 sweeps, residual), "
                         f"sweep.workers={cores}; factorization {s.factor_seconds:.2f}s excluded",
               "factor_seconds": s.factor_seconds, "seconds": dt}
        if u0 is not None:
            out["parity_rel_l2_rhs0"] = float(np.linalg.norm(u0 - u) / np.linalg.norm(u))
        return out
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "RHS/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle import ref
    base = {"impl": "reference", "metric": METRIC, "unit": "RHS/s", "higher_is_better": True,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "dtype": "c128",
            "data": "synthetic", "config": {"workload": WORKLOAD}}
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhelmsweep_ref.so not built"}))
        return 0
    cores = os.cpu_count() or 1
    s = ref.RefSolver(ref_config(), cores)
    f = make_sources(1000 + rank, s.lo, s.hi, s.hgrid, s.origin)
    B = [s.scale_source(f[r]) for r in range(CFG["nrhs"])]
    for w in range(args.warmup):
        s.ddm_solve(B[w % len(B)], CFG["rounds"], True)
    t0 = time.perf_counter()
    for k in range(args.steps):
        s.ddm_solve(B[k % len(B)], CFG["rounds"], True)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    base.update(value=v, ms_per_step=1e3 * dt / args.steps, scaling="weak", vs_baseline=None,
                cpu_baseline={"value": v, "unit": "RHS/s", "cores": cores, "kind": "reference",
                              "sample": f"{args.steps} RHS of the workload, one full DDM application each, "
                                        f"sweep.workers={cores}"},
                e2e={"value": v, "unit": "RHS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                factorization_seconds=s.factor_seconds)
    print(json.dumps(base))
    return 0


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2003_02585_b200 as hs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    setup = hs.ProblemSetup(2, [CFG["n"]] * 2, list(CFG["parts"]), hs.Medium("constant", kappa=CFG["kappa"]),
                            pml_width=CFG["pad"])
    # --partition subdomain (N > 1): one problem, its subdomains spread over the ranks (SURVEY.md
    # §8(e)); every rank solves the same 16 RHS -> strong scaling. Default: RHS sharding (weak).
    part = world > 1 and args.partition == "subdomain"
    t0 = time.perf_counter()
    if part:
        from paper_2003_02585_b200.multi import PartitionedDdmSolver
        s = PartitionedDdmSolver(setup, device=local_rank)
    else:
        s = hs.DdmSolver(setup, device=local_rank)
    setup_seconds = time.perf_counter() - t0
    N, R = s.global_n, CFG["nrhs"]
    units = R if part else R * world  # RHS the whole job completes per step
    hgrid = [1.0 / CFG["n"]] * 2
    f = make_sources(1000 + (0 if part else rank), s.lo, s.hi, hgrid, [0.0, 0.0])
    b = s.scale_source(f)  # (R, N) RHS-major
    db = torch.from_numpy(b.view(np.float64)).to(dev)
    du = torch.empty_like(db)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rounds, track = CFG["rounds"], True

    def step():
        s.ddm_solve_device(db.data_ptr(), du.data_ptr(), R, rounds, track, stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    L0 = hs.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize(dev)
    launches = hs.kernel_launches() - L0
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    prof = s.profile()  # solve-kernel profile of the last timed step (CUDA events on our stream)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = units / (ms_max * 1e-3)

    # e2e through the public API with pinned host buffers
    hb = torch.from_numpy(b.view(np.float64)).pin_memory()
    hu = torch.empty_like(hb).pin_memory()
    for _ in range(max(args.warmup, 3)):
        s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), R, rounds, track)
    if world > 1:
        dist.barrier()
    n_e2e = max(3, min(args.steps, 10))
    e2e_samples = []
    for _ in range(n_e2e):
        te = time.perf_counter()
        s.ddm_solve_host_ptr(hb.data_ptr(), hu.data_ptr(), R, rounds, track)
        e2e_samples.append(1e3 * (time.perf_counter() - te))
    e2e_ms = sum(e2e_samples) / n_e2e
    t2 = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_val = units / (float(t2.item()) * 1e-3)
    # parity sanity of what was timed: device result == host-path result
    ok = bool(torch.equal(du.cpu(), hu))

    if rank != 0:
        return 0
    hbm, hbm_kind, fp64 = peaks()
    sec = prof["solve_seconds"]
    tflops = prof["alg_flops"] / sec / 1e12
    gbs = prof["alg_bytes"] / sec / 1e9
    tr = ncu_traffic()
    nl = max(prof["solve_launches"], 1)
    line = {
        "metric": METRIC, "value": value, "unit": "RHS/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if part else "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": WORKLOAD, "rhs_per_gpu": R, "subdomains": s.nsub, "global_nodes": N,
                   "parallelism": (f"subdomain-partitioned x{world} (strong; NCCL trace/ghost exchange per macro-step)"
                                   if part else f"rhs-sharded x{world} (weak), subdomain steps batched per GPU"),
                   "l2": "inputs larger than L2 (2.5 GB resident factors streamed every step)"},
        # At 16 RHS the solve streams 16 B of factor per 8*16 flop: 8 flop/B > the 5.75 flop/B ridge
        # (37.1 TF FP64 DMMA / 6.46 TB/s), so the dominant kernels are FP64 tensor-core bound.
        "roofline": {"bound": "tensor", "achieved": tflops, "peak": fp64, "unit": "TFLOP/s", "frac": tflops / fp64,
                     "peak_source": "measured FP64 DMMA peak (profiles/fp64_peak.json, tools/bench_fp64.cu); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "traffic": tr.get("bytes_per_launch") if tr else None,
                     "kernel": "solve6_kernel<fwd|bwd> (multifrontal partitioned-inverse solve on DMMA, dataflow)",
                     "alg_flops_per_launch": prof["alg_flops"] / nl,
                     "alg_bytes_per_launch": prof["alg_bytes"] / nl,
                     "avg_launch_us": 1e6 * sec / nl,
                     "solve_share_of_step": sec / (ms_max * 1e-3),
                     "hbm_view": {"achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm,
                                  "peak_source": f"{hbm_kind} hbm_gbs (MEASURED_PEAKS.json)"}},
        "e2e": {"value": e2e_val, "unit": "RHS/s", "h2d_bytes_per_step": int(b.nbytes),
                "d2h_bytes_per_step": int(b.nbytes), "steps": n_e2e,
                "ms_per_step_samples": [round(x, 3) for x in e2e_samples]},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "factorization_seconds": s.factor_seconds(),
        "setup_seconds": setup_seconds,
        "sweep_seconds_per_rhs": ms_max * 1e-3 / R,
        "subdomain_solves_per_step": prof["subdomain_solves"],
        "device_host_paths_agree": ok,
    }
    if part:
        _, _, owned, sent, msgs = s.partition_info()
        line["partition"] = {"mode": "subdomain", "owned_subdomains_rank0": owned,
                             "exchange_bytes_per_application_rank0": 8 * sent, "messages_per_application_rank0": msgs}
    # The paper's pipeline cost model (src/pipeline.cpp) next to the device schedule: the model
    # runs one processor per subdomain, one RHS per tick; the device levels the same trace-routing
    # task graph into macro-steps and solves each task for the whole 16-RHS batch at once.
    sched = s.schedule_info(rounds)
    sim1 = hs.simulate_pipeline(2, list(CFG["parts"]), 1, rounds, 1.0)
    simR = hs.simulate_pipeline(2, list(CFG["parts"]), R, rounds, 1.0)
    line["pipeline_model"] = {
        "device_macro_steps": sched["macro_steps"], "device_max_width": sched["max_width"],
        "reference_sequential_steps": sched["sequential_steps"], "x_buffers": sched["buffers"],
        "model_ticks_1_rhs": sim1.makespan, f"model_ticks_{R}_rhs": simR.makespan,
        "model_closed_form_ticks_per_rhs": hs.average_time_per_rhs(2, list(CFG["parts"]), R, rounds, 1.0).average_per_rhs,
        "device_t0_us_per_16rhs_task": 1e6 * prof["solve_seconds"] / max(prof["subdomain_solves"], 1),
        "device_ms_per_macro_step": ms_max / max(sched["macro_steps"], 1)}
    if world == 1 and not args.no_cpu_baseline:
        u0 = hu[0].numpy().view(np.complex128) if hu.dim() > 1 else None
        line["cpu_baseline"] = cpu_baseline_sample(b[0], u0)
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partition", default="rhs", choices=["rhs", "subdomain"],
                    help="multi-GPU layout: RHS sharding (weak scaling) or subdomain partitioning (strong)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
