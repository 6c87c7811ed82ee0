"""Summarise this round's evidence job (tools/evidence_job.sh, merged into gpurun_out/) into
profiles/: the bench line, per-kernel totals and DRAM throughput of the ncu launch list, and the
ncu --set full metrics of the solve and sweep kernels.  python tools/profiles_r2.py"""
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    iK, iM, iV, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    k = collections.defaultdict(dict)
    for r in data:
        if len(r) < len(hdr):
            continue
        k[r[iID]]["name"] = r[iK]
        k[r[iID]][r[iM]] = float(r[iV].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for d in k.values():
        n = d["name"].split("(")[0].replace("void ", "").replace("hsb::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
        a = agg[n]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0)
        a[3] += d.get("dram__bytes_write.sum", 0)
    return agg


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = []
    want = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "read", "dram__bytes_write.sum": "write",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
            "launch__registers_per_thread": "regs"}
    units = rows[1]
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m, key in want.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    x = float(v)
                except ValueError:
                    continue
                if key == "us":
                    x = x / 1e3 if u == "ns" else x * 1e3 if u == "ms" else x
                if key in ("read", "write"):
                    x *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)
                d[key] = x
        if "us" in d and "read" in d:
            d["dram_gbs"] = (d["read"] + d.get("write", 0)) / (d["us"] * 1e-6) / 1e9
        res.append(d)
    return res


def compact_launch_list(src, dst):
    """Per-launch list (id, kernel, ns, DRAM read / write bytes) of the ncu metrics pass."""
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    iK, iM, iV, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    k = collections.OrderedDict()
    for r in data:
        if len(r) < len(hdr):
            continue
        d = k.setdefault(r[iID], {})
        d["name"] = (r[iK].split("(")[0].replace("void ", "").replace("hsb::", "").replace("<unnamed>::", "")
                     .replace("unnamed>::", ""))
        d[r[iM]] = float(r[iV].replace(",", ""))
    L = [(d["name"], int(d.get("gpu__time_duration.sum", 0)), int(d.get("dram__bytes_read.sum", 0)),
          int(d.get("dram__bytes_write.sum", 0))) for d in k.values()]
    with open(dst, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none  "
                "python bench.py --steps 1 --warmup 3 --no-cpu-baseline (C3, 64 RHS)\n")
        f.write("id,kernel,duration_ns,dram_read_bytes,dram_write_bytes\n")
        for i, x in enumerate(L):
            f.write(f"{i},{x[0]},{x[1]},{x[2]},{x[3]}\n")
    return L


def application_traffic(L, bench, full):
    """DRAM bytes of the solve launches of the timed device application (the 4th: after 3 warm-ups)
    against the same application's algorithmic bytes -> profiles/solve_traffic.json (bench.py's
    roofline.traffic)."""
    starts = [i for i, x in enumerate(L) if x[0].startswith("transpose_in_kernel")]
    ends = [i for i, x in enumerate(L) if x[0].startswith("transpose_out_kernel")]
    sv = [x for x in L[starts[3]:ends[3]] if x[0].startswith("solve6")]
    tot, t = sum(x[2] + x[3] for x in sv), sum(x[1] for x in sv)
    alg = bench["roofline"]["alg_bytes_per_launch"] * len(sv)
    out = {"what": "ncu dram__bytes_read + write summed over the solve launches of the timed 64-RHS C3 application "
                   "(profiles/r2_launch_list.csv), per launch, against the same application's algorithmic bytes",
           "bytes_per_launch": tot / len(sv), "launches": len(sv), "dram_bytes_application": tot,
           "alg_bytes_application": alg, "dram_over_algorithmic": tot / alg, "ncu_serialised_ms": t / 1e6,
           "dram_gbs_under_ncu": tot / t, "full_capture_step35": full}
    json.dump(out, open(os.path.join(P, "solve_traffic.json"), "w"), indent=1)
    return out


def main():
    lines = []
    bench = open(os.path.join(G, "r2_bench.log")).read().strip().splitlines()[-1]
    b = json.loads(bench)
    json.dump(b, open(os.path.join(P, "r2_bench.json"), "w"), indent=1)
    lines += ["# Profile summary r2 (B200, C3 workload, 64 RHS)", "",
              f"Bench (`r2_bench.json`): {b['value']:.1f} RHS/s device ({b['ms_per_step']:.1f} ms per 64-RHS application), "
              f"e2e {b['e2e']['value']:.1f} RHS/s, solve kernels {b['roofline']['achieved']:.2f} TF/s = "
              f"{100 * b['roofline']['frac']:.1f}% of the FP64 DMMA peak; CPU reference "
              f"{b['cpu_baseline']['value']:.3f} RHS/s on {b['cpu_baseline']['cores']} cores; parity "
              f"{b['cpu_baseline'].get('parity_rel_l2_rhs0')}", ""]
    agg = launch_list(os.path.join(G, "r2_launches.csv"))
    tot = sum(a[1] for a in agg.values())
    lines += ["Launch list (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
              "--clock-control none` over `bench.py --steps 1 --warmup 3 --no-cpu-baseline`: setup, 3 warm-up, 1 "
              "timed and the e2e applications; per-launch times are cold-cache and serialised):", "",
              "| kernel | launches | total ms | share | us / launch | DRAM GB/s | % of 6548 GB/s |", "|---|---|---|---|---|---|---|"]
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:22]:
        gbs = (a[2] + a[3]) / a[1] if a[1] else 0.0
        lines.append(f"| `{n}` | {a[0]} | {a[1] / 1e6:.2f} | {100 * a[1] / tot:.1f}% | {a[1] / a[0] / 1e3:.1f} | "
                     f"{gbs:.0f} | {100 * gbs / 6548.5:.0f}% |")
    with open(os.path.join(P, "r2_launch_totals.json"), "w") as f:
        json.dump({n: {"launches": a[0], "ms": a[1] / 1e6, "dram_bytes": a[2] + a[3]} for n, a in agg.items()}, f, indent=1)
    for rep, title in (("r2_solve_full.ncu-rep", "solve kernels, C3 macro-step 35 (31 tasks x 64 RHS)"),
                       ("r2_sweep_full.ncu-rep", "sweep kernels, C3"),
                       ("r2_acc_full.ncu-rep", "column order, transposes, fused accumulate, residual, C3")):
        path = os.path.join(G, rep)
        if not os.path.exists(path):
            continue
        fm = full_metrics(path)
        lines += ["", f"Full capture ({title}, `ncu --set full`):", "",
                  "| kernel | us | DRAM MB | DRAM GB/s | DRAM % | DMMA pipe % | warps active % | regs |", "|---|---|---|---|---|---|---|---|"]
        for d in fm:
            lines.append(f"| `{d['kernel']}` | {d.get('us', 0):.1f} | {(d.get('read', 0) + d.get('write', 0)) / 1e6:.0f} | "
                         f"{d.get('dram_gbs', 0):.0f} | {d.get('dram_pct', 0):.0f} | {d.get('dmma_pct', 0):.1f} | "
                         f"{d.get('warps_active_pct', 0):.1f} | {d.get('regs', 0):.0f} |")
        if rep.startswith("r2_solve"):
            sv = [d for d in fm if "solve6" in d["kernel"]]
            full = {"what": "ncu --set full DRAM bytes per solve launch (C3 macro-step 35, fwd + bwd average)",
                    "bytes_per_launch": sum(d.get("read", 0) + d.get("write", 0) for d in sv) / max(len(sv), 1),
                    "launches": sv}
            L = compact_launch_list(os.path.join(G, "r2_launches.csv"), os.path.join(P, "r2_launch_list.csv"))
            tr = application_traffic(L, b, full)
            lines += ["", f"Solve launches of the timed application: {tr['dram_bytes_application'] / 1e9:.0f} GB of DRAM traffic "
                      f"against {tr['alg_bytes_application'] / 1e9:.0f} GB algorithmic = {tr['dram_over_algorithmic']:.2f}x "
                      f"(`solve_traffic.json`)."]
    open(os.path.join(P, "r2_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
