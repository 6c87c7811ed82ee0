"""Developer run of BASELINE configs 3 and 4 on one B200, with parity against the reference
(oracle/_ref, the reference compiled in place, timed on the box's host cores).

  python tools/run_config.py c3 [--ref-full]   2048^2 two-layered, 16x16, 2 rounds, 64 RHS
  python tools/run_config.py c4 [--ref-small]  4096^2 GRF medium, 32x32, GMRES(30) to 1e-8, 32 RHS

c3: the GPU solves all 64 RHS (two 32-RHS batches); --ref-full runs the reference on RHS 0 at
full scale (factorization + one DDM application) and compares u (<= 1e-9) and the counters.
c4: the GPU runs GMRES for all 32 RHS in memory-sized batches; --ref-small runs the reference
and the GPU on the same medium and subdomain size at a reduced partition (8x8 subdomains of
209^2, grid 1024^2: SURVEY.md §8(d) "run parity on a reduced geometry with the same subdomain
size") and compares one DDM application (<= 1e-9) and GMRES iteration counts (+-1).
Writes gpurun_out/<cfg>.json."""
import argparse, json, math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2003_02585_b200 as hs
from paper_2003_02585_b200 import sources

OUT = os.path.join(ROOT, "gpurun_out")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def srcs(s, n, count, seed):
    return sources.gaussian_sources(2, s.lo, s.hi, [1.0 / n] * 2, [0.0, 0.0], sources.seeded_centers(seed, count, 2),
                                    2.0 / n)


def c3(args, out):
    n, parts, pad, R, rounds = 2048, 16, 32, 64, 2
    kd, ku, eta = 2 * math.pi * 96, 2 * math.pi * 64, 0.5 + 1.0 / 4096
    med = hs.Medium("two_layered", kappa_down=kd, kappa_up=ku, axis=1, eta=eta, eps=0.0)
    t = time.perf_counter()
    s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [parts, parts], med, pml_width=pad))
    out.update(config="C3: 2D two-layered (c=1 / 1.5 at y=0.5+h/2), 2048^2 + 32 PML, 16x16, omega=2pi*96, "
                      "2 rounds, 64 RHS", setup_seconds=time.perf_counter() - t, factor_seconds=s.factor_seconds(),
               global_nodes=s.global_n)
    b = s.scale_source(srcs(s, n, R, 3000))
    s.ddm_solve(b[:32], rounds, [], True)  # warm-up (buffers, plans)
    reps = []
    t = time.perf_counter()
    U = s.ddm_solve(b, rounds, reps, True)
    wall = time.perf_counter() - t
    dev = reps[0].sweep_seconds_total + reps[32].sweep_seconds_total
    out.update(rhs=R, device_seconds=dev, rhs_per_s_device=R / dev, wall_seconds_host_buffers=wall,
               rhs_per_s_e2e=R / wall, local_solves_rhs0=reps[0].local_solves,
               skipped_rhs0=reps[0].skipped_zero_solves, round_residuals_rhs0=reps[0].round_residuals)
    print(json.dumps(out), flush=True)
    if args.ref_full:
        from oracle import ref
        cfg = {"dim": 2, "grid.n": [n, n], "partition": [parts, parts], "pml.width": pad, "media.kind": "two_layered",
               "media.kappa_down": kd, "media.kappa_up": ku, "media.axis": 1, "media.eta_L": eta,
               "media.epsilon": 0.0}
        cores = os.cpu_count()
        r = ref.RefSolver(cfg, cores)
        u0, rep0 = r.ddm_solve(b[0], rounds, True)
        keys = ["traces_generated", "traces_routed", "traces_discarded", "local_solves", "skipped_zero_solves"]
        out.update(ref_cores=cores, ref_factor_seconds=r.factor_seconds,
                   ref_sweep_seconds_rhs0=rep0["sweep_seconds_total"], ref_rhs_per_s=1.0 / rep0["sweep_seconds_total"],
                   rel_l2_vs_reference_rhs0=rel(U[0], u0),
                   counters_equal=[getattr(reps[0], k) for k in keys] == [rep0[k] for k in keys],
                   round_residuals_ref=rep0["round_residuals"])
    return out


def c4_medium(n_lattice=4096, seed=2024):
    c = sources.gaussian_random_velocity(n_lattice, seed)
    return c, hs.Medium("gridded", velocity=c.ravel(), vel_n=(n_lattice + 1, n_lattice + 1, 1),
                        vel_origin=(0.0, 0.0, 0.0), vel_spacing=(1.0 / n_lattice, 1.0 / n_lattice, 0.0),
                        omega=2 * math.pi * 160)


def c4(args, out):
    pad, R, tol, maxit, restart = 40, 32, 1e-8, 250, 30
    c, med = c4_medium()
    out.update(config="C4: 2D GRF medium c=1+0.5(1+tanh g)/2 (corr. 0.05, seed 2024), 4096^2 + 40 PML, 32x32, "
                      "omega=2pi*160, GMRES(30) to 1e-8 (<= 250 iterations) with the DDM preconditioner, 32 RHS",
               velocity_min=float(c.min()), velocity_max=float(c.max()))
    if not args.skip_full:
        n = 4096
        t = time.perf_counter()
        s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [32, 32], med, pml_width=pad))
        out.update(setup_seconds=time.perf_counter() - t, factor_seconds=s.factor_seconds(), global_nodes=s.global_n)
        print(json.dumps(out), flush=True)
        b = s.scale_source(srcs(s, n, R, 4000))
        t = time.perf_counter()
        G = s.gmres(b, tol, maxit, 1, restart=restart)  # GMRES(30), up to 250 iterations
        wall = time.perf_counter() - t
        its = [g.iterations for g in G]
        out.update(rhs=R, gmres_seconds=wall, rhs_per_s=R / wall, iterations=its,
                   converged=all(g.converged for g in G), max_true_residual=max(g.true_residual for g in G))
        print(json.dumps(out), flush=True)
        del s
    if args.ref_full:
        # SURVEY.md §8(d) C4 pin at full scale (32x32 subdomains of 209^2, 4096^2 + 40 PML): one DDM
        # application's per-round residual and u, then 30 GMRES iterations (the reference's gmres is
        # unrestarted, so its first 30 iterations are GMRES(30)'s first cycle) for one RHS, on the
        # GPU and on the reference (oracle/_ref, all host cores)
        from oracle import ref
        n = 4096
        path = "/tmp/c4_velocity_full.hsvg"
        hs.write_velocity_grid(path, hs.VelocityGrid(2, [4097, 4097, 1], [0.0, 0.0, 0.0], [1 / 4096, 1 / 4096, 0.0],
                                                     c.ravel()))
        s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [32, 32], med, pml_width=pad))
        b = s.scale_source(srcs(s, n, 1, 4000))
        reps = []
        U = s.ddm_solve(b, 1, reps, True)
        G = s.gmres(b, tol, 30, 1, restart=30)
        full = {"geometry": "full C4: 4096^2 + 40 PML, 32x32 subdomains of 209^2", "gpu_round_residual": reps[0].round_residuals,
                "gpu_gmres_iterations": G[0].iterations, "gpu_history": G[0].history}
        print(json.dumps(full), flush=True)
        cores = os.cpu_count()
        t = time.perf_counter()
        r = ref.RefSolver({"dim": 2, "grid.n": [n, n], "partition": [32, 32], "pml.width": pad, "media.kind": "gridded",
                           "media.velocity_file": path, "media.omega": 2 * math.pi * 160}, cores)
        full["ref_factor_seconds"] = time.perf_counter() - t
        br = r.scale_source(srcs(s, n, 1, 4000)[0])
        full["rhs_bitwise_equal"] = bool(np.array_equal(b[0], br))
        t = time.perf_counter()
        u0, rep0 = r.ddm_solve(br, 1, True)
        full.update(ref_application_seconds=time.perf_counter() - t, ref_round_residual=rep0["round_residuals"],
                    ddm_rel_l2_vs_reference=rel(U[0], u0),
                    counters_equal=[getattr(reps[0], k) for k in ("local_solves", "skipped_zero_solves", "traces_routed",
                                                                    "traces_discarded")] ==
                    [rep0[k] for k in ("local_solves", "skipped_zero_solves", "traces_routed", "traces_discarded")])
        print(json.dumps(full), flush=True)
        xr, gr = r.gmres(br, tol, 30, 1)
        h_gpu, h_ref = np.array(G[0].history), np.array(gr["history"])
        k = min(len(h_gpu), len(h_ref))
        full.update(ref_gmres_iterations=gr["iterations"], ref_history=gr["history"], ref_gmres_seconds=gr["seconds"],
                    history_max_rel_diff=float(np.max(np.abs(h_gpu[:k] - h_ref[:k]) / np.abs(h_ref[:k]))),
                    gmres_x_rel_l2=rel(G[0].x, xr), ref_cores=cores)
        out["full_parity"] = full
    if args.ref_small:
        from oracle import ref
        n = 1024
        path = "/tmp/c4_velocity.hsvg"  # 64 MB: kept out of gpurun_out
        hs.write_velocity_grid(path, hs.VelocityGrid(2, [4097, 4097, 1], [0.0, 0.0, 0.0], [1 / 4096, 1 / 4096, 0.0],
                                                     c.ravel()))
        s = hs.DdmSolver(hs.ProblemSetup(2, [n, n], [8, 8], med, pml_width=pad))
        cfg = {"dim": 2, "grid.n": [n, n], "partition": [8, 8], "pml.width": pad, "media.kind": "gridded",
               "media.velocity_file": path, "media.omega": 2 * math.pi * 160}
        cores = os.cpu_count()
        r = ref.RefSolver(cfg, cores)
        b = s.scale_source(srcs(s, n, 2, 4100))
        br = np.stack([r.scale_source(srcs(s, n, 2, 4100)[i]) for i in range(2)])
        reps = []
        U = s.ddm_solve(b, 1, reps, True)
        small = {"geometry": "1024^2 + 40 PML, 8x8 subdomains of 209^2 (C4's subdomain size), same medium/omega",
                 "rhs_bitwise_equal": bool(np.array_equal(b, br))}
        u0, rep0 = r.ddm_solve(br[0], 1, True)
        small["ddm_rel_l2_vs_reference"] = rel(U[0], u0)
        G = s.gmres(b, tol, 60, 1)  # the reference's full GMRES (gmres.maxit default 60)
        gi = []
        for i in range(2):
            xr, gr = r.gmres(br[i], tol, 60, 1)
            gi.append({"gpu_iterations": G[i].iterations, "ref_iterations": gr["iterations"],
                       "x_rel_l2": rel(G[i].x, xr), "ref_seconds": gr["seconds"]})
        small.update(gmres=gi, ref_cores=cores, ref_factor_seconds=r.factor_seconds)
        out["reduced_parity"] = small
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", choices=["c3", "c4"])
    ap.add_argument("--ref-full", action="store_true")
    ap.add_argument("--ref-small", action="store_true")
    ap.add_argument("--skip-full", action="store_true")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    out = {}
    out = c3(args, out) if args.cfg == "c3" else c4(args, out)
    print(json.dumps(out), flush=True)
    with open(os.path.join(OUT, f"{args.cfg}.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
