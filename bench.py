"""Benchmark: RHS/s through full 2^n diagonal sweeps (BASELINE.json metric) on B200.

Headline workload (BASELINE.json configs[2], "C3" -- the largest single-GPU configuration; C5 is
the 8-GPU configuration and C4 is GMRES mode): 2D two-layered medium, 2048^2 interior + 32-cell
PML, c = 1 below y = 0.5 + h/2 and 1.5 above (omega = 2 pi 96 referenced to c = 1), 16x16
checkerboard subdomains each with its own 32-cell PML, 64 RHS = Gaussian point sources (sigma = 2h,
unit amplitude) at seeded uniform interior locations, complex128, direct-solver mode: one DDM
application = 2 rounds of 4 diagonal sweeps with the per-round residual the reference's
run_direct tracks (src/harness.cpp:269-283). ``--config c2`` runs BASELINE configs[1] (1024^2,
8x8, 16 RHS, 1 round) instead.

A step is one DDM application over the batch of RHS (lockstep-batched through every subdomain
solve). ``value`` = RHS/s with b already resident in HBM, device-timed with CUDA events;
``e2e`` = the same through hs_ddm_solve with pinned host buffers (H2D of b and D2H of u inside
the timed region). Multi-GPU (torchrun): one process per GPU, each rank sweeps its own RHS batch
against its own resident factors (RHS are independent units; no data-path collective) -> weak
scaling, time = max over ranks, with ``--partition rhs``; the default for N > 1 spreads one
problem's subdomains over the ranks (BASELINE north_star) with the library's own
NCCL transport (hs_ddm_create_nccl) -> strong scaling.

``--impl reference`` runs the reference's own CPU implementation (oracle/_ref, the unmodified
reference compiled in place) on the host cores, one RHS per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RHS/sec through full 2^n diagonal sweeps"
CONFIGS = {
    "c3": dict(
        workload=("C3: 2D two-layered medium (c=1 for y<0.5+h/2, c=1.5 above), 2048^2 grid + 32-cell PML, "
                  "omega=2pi*96 (c=1), 16x16 subdomains, 64 RHS seeded Gaussian sources (sigma=2h), direct-solver "
                  "mode (2 rounds = 8 diagonal sweeps, per-round residual)"),
        dim=2, n=2048, parts=(16, 16), pad=32, nrhs=64, rounds=2, kind="two_layered",
        kappa_down=2 * math.pi * 96, kappa_up=2 * math.pi * 64, eta=0.5 + 1.0 / 4096, seed=3000),
    "c2": dict(
        workload=("C2: 2D constant medium c=1, 1024^2 grid + 32-cell PML, omega=2pi*64, 8x8 subdomains, "
                  "16 RHS seeded Gaussian sources (sigma=2h), direct-solver mode (1 round = 4 diagonal sweeps, "
                  "per-round residual)"),
        dim=2, n=1024, parts=(8, 8), pad=32, nrhs=16, rounds=1, kind="constant", kappa=2 * math.pi * 64, seed=1000),
}
CFG = dict(CONFIGS["c3"])
WORKLOAD = CFG["workload"]


def select(name):
    global WORKLOAD
    CFG.clear()
    CFG.update(CONFIGS[name])
    WORKLOAD = CFG["workload"]


def ref_config():
    c = {"dim": 2, "grid.n": [CFG["n"]] * 2, "partition": list(CFG["parts"]), "pml.width": CFG["pad"]}
    if CFG["kind"] == "constant":
        c.update({"media.kind": "constant", "media.kappa": CFG["kappa"]})
    else:
        c.update({"media.kind": "two_layered", "media.kappa_down": CFG["kappa_down"],
                  "media.kappa_up": CFG["kappa_up"], "media.axis": 1, "media.eta_L": CFG["eta"],
                  "media.epsilon": 0.0})
    return c


def medium(hs):
    if CFG["kind"] == "constant":
        return hs.Medium("constant", kappa=CFG["kappa"])
    return hs.Medium("two_layered", kappa_down=CFG["kappa_down"], kappa_up=CFG["kappa_up"], axis=1,
                     eta=CFG["eta"], eps=0.0)


def host_info():
    """CPU model, core count and RAM of the host the CPU baseline ran on."""
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    ram = round(int(line.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    try:  # the shim's large dense products run on numpy's bundled OpenBLAS when it loads (oracle/shim)
        from oracle import ref
        dense = ("large dense products on numpy's bundled OpenBLAS, one thread per worker" if ref.blas_active()
                 else "naive dense loops, no BLAS")
    except Exception:
        dense = "dense backing unknown"
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gib": ram,
            "reference_build": "g++ -O3 -march=native, reference sources compiled in place against the "
                               f"from-scratch Eigen-subset shim oracle/shim ({dense})"}


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


def hbm_bound_companion():
    """The same solve kernels where they are HBM-bound (8 RHS: 4 flop per factor byte, below the
    5.7 flop/B ridge): the committed C5 run (tools/check_c5.py -> profiles/r2_c5.json), not measured
    by this command."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2_c5.json")) as f:
            c = json.load(f)["solve"]
        return {"config": "C5 (3D, 64 subdomains of 57^3, 8 RHS)", "achieved_gbs": c["achieved_gbs"],
                "frac": c["hbm_frac"], "source": "profiles/r2_c5.json (tools/check_c5.py; not measured by this run)"}
    except Exception:
        return None


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
    every subdomain, then one RHS of the workload through one DDM application. With u0 (the
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
               "sample": f"1 of the {CFG['nrhs']} RHS through one full DDM application "
                         f"({4 * CFG['rounds']} sweeps, residual), sweep.workers={cores}; factorization "
                         f"{s.factor_seconds:.2f}s excluded",
               "factor_seconds": s.factor_seconds, "seconds": dt, "host": host_info(),
               "counters": {k: rep[k] for k in ("local_solves", "skipped_zero_solves", "traces_generated",
                                                "traces_routed", "traces_discarded")}}
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
    f = make_sources(CFG["seed"], s.lo, s.hi, s.hgrid, s.origin)
    B = [s.scale_source(f[r]) for r in range(min(CFG["nrhs"], args.warmup + args.steps))]
    del f
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
                                        f"sweep.workers={cores}", "host": host_info()},
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
    setup = hs.ProblemSetup(2, [CFG["n"]] * 2, list(CFG["parts"]), medium(hs), pml_width=CFG["pad"])
    # --partition subdomain (N > 1): one problem, its subdomains spread over the ranks (SURVEY.md
    # §8(e)); every rank solves the same RHS batch -> strong scaling. Default: RHS sharding (weak).
    part = world > 1 and args.partition == "subdomain"
    t0 = time.perf_counter()
    if part:
        from paper_2003_02585_b200.multi import make_partitioned
        s = make_partitioned(setup, device=local_rank)  # native NCCL transport inside the library
    else:
        s = hs.DdmSolver(setup, device=local_rank)
    setup_seconds = time.perf_counter() - t0
    N, R = s.global_n, CFG["nrhs"]
    units = R if part else R * world  # RHS the whole job completes per step
    hgrid = [1.0 / CFG["n"]] * 2
    f = make_sources(CFG["seed"] + (0 if part else rank), s.lo, s.hi, hgrid, [0.0, 0.0])
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
    # parity sanity of what was timed: device result vs host-path result. The device call runs one
    # R-RHS batch, the host-buffer call streams 32-RHS batches whose split-K shape differs, so the
    # two agree to roundoff (bitwise only when the batch widths coincide).
    duh = du.cpu()
    bitwise = bool(torch.equal(duh, hu))
    path_diff = float(torch.linalg.vector_norm(duh - hu) / torch.linalg.vector_norm(duh))
    del duh
    reps0 = s.ddm_solve_device(db.data_ptr(), du.data_ptr(), R, rounds, track, stream, want_reports=True)

    if rank != 0:
        return 0
    hbm, hbm_kind, fp64 = peaks()
    fac_gb = s.factor_bytes() / 1e9
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
                   "l2": f"inputs larger than L2 ({fac_gb:.1f} GB resident factors streamed every step, "
                         f"126 MB L2)"},
        # A batch of R RHS streams 16 B of factor per 8*R flop per pass: at R >= 16 that is >= 8 flop/B,
        # above the 5.75 flop/B ridge (37.1 TF FP64 DMMA / 6.46 TB/s), so the dominant kernels are FP64
        # tensor-core bound. `achieved` counts effective complex flops (8 real flops per complex
        # multiply-add of the algorithm); with the 3M products the pipe executes 6 real
        # flops per complex MAC on 8x8-block-padded tiles (pipe_view).
        "roofline": {"bound": "tensor", "achieved": tflops, "peak": fp64, "unit": "TFLOP/s", "frac": tflops / fp64,
                     "flops": "effective complex flops (8 per complex MAC of the packed factor, work performed: the RHS "
                              "columns the items computed -- RHS groups that are exactly zero for a task are skipped, as "
                              "the reference skips exact-zero solves, and are not counted)",
                     "peak_source": "measured FP64 DMMA peak (profiles/fp64_peak.json, tools/bench_fp64.cu); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "pipe_view": {"real_flops_per_complex_mac": 6 if prof.get("m3", True) else 8,
                                   "note": "pipe flops = achieved x 6/8 (3M) x block padding; ncu DMMA pipe-active "
                                           "share in profiles/"},
                     "traffic": tr.get("bytes_per_launch") if tr else None,
                     "kernel": "solve6_kernel<fwd|bwd> (multifrontal partitioned-inverse solve on DMMA, dataflow)",
                     "alg_flops_per_launch": prof["alg_flops"] / nl,
                     "alg_bytes_per_launch": prof["alg_bytes"] / nl,
                     "avg_launch_us": 1e6 * sec / nl,
                     "solve_share_of_step": sec * s.batches_per_application(R) / (ms_max * 1e-3),
                     "hbm_view": {"achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm,
                                  "peak_source": f"{hbm_kind} hbm_gbs (MEASURED_PEAKS.json)",
                                  "hbm_bound_regime": hbm_bound_companion()}},
        "e2e": {"value": e2e_val, "unit": "RHS/s", "h2d_bytes_per_step": int(b.nbytes),
                "d2h_bytes_per_step": int(b.nbytes), "steps": n_e2e,
                "ms_per_step_samples": [round(x, 3) for x in e2e_samples]},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "factorization_seconds": s.factor_seconds(),
        "setup_seconds": setup_seconds,
        "sweep_seconds_per_rhs": ms_max * 1e-3 / R,
        "subdomain_solves_per_step": prof["subdomain_solves"],
        "device_host_paths_agree": path_diff <= 1e-11,
        "device_host_paths_rel_l2": path_diff,
        "device_host_paths_bitwise": bitwise,
    }
    if part:
        _, _, owned, sent, msgs = s.partition_info()
        line["partition"] = {"mode": "subdomain", "owned_subdomains_rank0": owned,
                             "exchange_bytes_per_application_rank0": 8 * sent, "messages_per_application_rank0": msgs}
    # The paper's pipeline cost model (src/pipeline.cpp:20-111) against the
    # measured application. The model runs one processor per subdomain and one
    # unit of work per tick; on the device the unit is one RHS batch (every task of a macro-step runs
    # concurrently, the batch's RHS in lockstep), so T0 = the measured device time of one macro-step's
    # solve launches and the model's makespan for `batches` units predicts the application time.
    sched = s.schedule_info(rounds)
    parts = list(CFG["parts"])
    batches = s.batches_per_application(R)
    t0 = sec / max(nl / 2, 1)  # seconds per macro-step (forward + backward launch), last batch
    sim1 = hs.simulate_pipeline(2, parts, 1, rounds, 1.0)
    simB = hs.simulate_pipeline(2, parts, batches, rounds, t0)
    line["pipeline_model"] = {
        "device_macro_steps": sched["macro_steps"], "device_max_width": sched["max_width"],
        "reference_sequential_steps": sched["sequential_steps"], "x_buffers": sched["buffers"],
        "model_ticks_1_unit": sim1.makespan, "batches_per_application": batches,
        "t0_ms_per_macro_step_measured": 1e3 * t0,
        "model_predicted_solve_ms": 1e3 * simB.makespan,
        "model_closed_form_ms_per_batch": 1e3 * hs.average_time_per_rhs(2, parts, batches, rounds, t0).average_per_rhs,
        "measured_ms_per_application": ms_max,
        "measured_solve_ms_per_application": 1e3 * sec * batches,
        "predicted_over_measured": simB.makespan / (ms_max * 1e-3)}
    if world == 1 and not args.no_cpu_baseline:
        u0 = hu[0].numpy().view(np.complex128) if hu.dim() > 1 else None
        cb = cpu_baseline_sample(b[0], u0)
        if "counters" in cb:
            keys = list(cb["counters"])
            cb["counters_equal_rhs0"] = {k: getattr(reps0[0], k) for k in keys} == cb["counters"]
            cb["round_residuals_rhs0_gpu"] = reps0[0].round_residuals
        line["cpu_baseline"] = cb
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS),
                    help="BASELINE configuration: c3 (configs[2], the headline) or c2 (configs[1])")
    ap.add_argument("--partition", default="subdomain", choices=["rhs", "subdomain"],
                    help="multi-GPU layout (N > 1): subdomain partitioning over the ranks with the library's "
                         "native NCCL trace exchange (strong scaling, BASELINE north_star) or RHS sharding (weak)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    select(args.config)
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
