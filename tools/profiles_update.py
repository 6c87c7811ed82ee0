"""Regenerate profiles/ from a gpurun evidence job (tools/gpujob_r1.sh) merged into gpurun_out/:
the bench line, the compact ncu launch list with per-kernel totals, and the full-capture summary
with per-launch DRAM traffic of the solve kernels (profiles/solve_traffic.json, which bench.py
reports as roofline.traffic)."""
import collections, csv, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"


def us(d):
    v = float(d["Metric Value"].replace(",", ""))
    return {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[d["Metric Unit"]]


def main():
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(os.path.join(OUT, f"bench_{tag}.json"), os.path.join(PROF, f"{tag}_bench.json"))
    rows = list(csv.reader(open(os.path.join(OUT, f"launches_{tag}.csv"))))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    with open(os.path.join(PROF, f"{tag}_launch_list.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "duration_us"])
        for d in data:
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            w.writerow([d["ID"], k, d["Grid Size"], d["Block Size"], round(us(d), 3)])
            agg[k][0] += 1
            agg[k][1] += us(d)
    raw = subprocess.run(["ncu", "-i", os.path.join(OUT, f"solve_full_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h = rr[0]

    def g(r, n):
        i = h.index(n)
        return float(r[i]) if r[i] else None
    caps = []
    for r in rr[2:]:
        caps.append({"kernel": r[h.index("Kernel Name")], "duration_us": g(r, "gpu__time_duration.sum"),
                     "dram_read_MB": g(r, "dram__bytes_read.sum"), "dram_write_MB": g(r, "dram__bytes_write.sum"),
                     "dmma_pipe_active_pct": g(r, "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
                     "sm_throughput_pct": g(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "warps_active_pct": g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                     "registers": g(r, "launch__registers_per_thread"), "grid": g(r, "launch__grid_size")})
    traffic = [c["dram_read_MB"] + c["dram_write_MB"] for c in caps]
    out = {"source": f"ncu --set full --clock-control none, tools/prof_step.py (C2, 16 RHS), solve6 launches 29-30 "
                     f"= the forward and backward launch of macro-step 14 (15 tasks), {tag}",
           "bytes_per_launch": 1e6 * sum(traffic) / len(traffic), "launches": caps}
    # every solve launch of one application (ncu --metrics dram__bytes_*), comparable with the bench's
    # alg_bytes_per_launch, which averages over the same launches
    allp = os.path.join(OUT, "solve_dram_all.csv")
    if os.path.exists(allp):
        per = collections.defaultdict(float)
        rows = list(csv.reader(open(allp)))
        hdr = None
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d["Metric Name"].startswith("dram__bytes"):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["Metric Unit"]]
                    per[d["ID"]] += float(d["Metric Value"].replace(",", "")) * scale
        out["source_all_launches"] = (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                                      f"over all {len(per)} solve launches of one C2 application (tools/prof_step.py)")
        out["bytes_per_launch"] = sum(per.values()) / max(len(per), 1)
        out["bytes_per_launch_macro_step_14"] = 1e6 * sum(traffic) / len(traffic)
    json.dump(out, open(os.path.join(PROF, "solve_traffic.json"), "w"), indent=1)
    bench = json.load(open(os.path.join(PROF, f"{tag}_bench.json")))
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write(f"# Profile summary {tag} (B200, C2 workload, 16 RHS)\n\n")
        f.write(f"Bench line: `{tag}_bench.json` — value {bench['value']:.1f} RHS/s ({bench['ms_per_step']:.2f} ms per "
                f"application), e2e {bench['e2e']['value']:.1f} RHS/s, solve kernels {bench['roofline']['achieved']:.2f} "
                f"TFLOP/s = {100 * bench['roofline']['frac']:.1f}% of the measured FP64 DMMA peak, CPU reference "
                f"{bench['cpu_baseline']['value']:.3f} RHS/s on {bench['cpu_baseline']['cores']} cores.\n\n")
        f.write("Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` over `python bench.py --steps 1 "
                "--warmup 3 --no-cpu-baseline` (setup + 3 warm-up + 1 timed + 2 e2e applications; per-launch times are "
                f"cold-cache and serialised). Raw list: `{tag}_launch_list.csv`.\n\n")
        f.write("| kernel | launches | total ms | per launch us | share |\n|---|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{k}` | {v[0]} | {v[1] / 1e3:.2f} | {v[1] / v[0]:.1f} | {100 * v[1] / tot:.1f}% |\n")
        f.write(f"\nFull capture (`ncu --set full`, `solve_full_{tag}.ncu-rep`, not committed): macro-step 14 "
                "(15 tasks x 16 RHS).\n\n")
        f.write("| kernel | us | DRAM read MB | DRAM write MB | DMMA pipe active % | warps active % |\n|---|---|---|---|---|---|\n")
        for c in caps:
            f.write(f"| `{c['kernel']}` | {c['duration_us']:.1f} | {c['dram_read_MB']:.0f} | {c['dram_write_MB']:.0f} | "
                    f"{c['dmma_pipe_active_pct']:.1f} | {c['warps_active_pct']:.1f} |\n")
    print(open(os.path.join(PROF, f"{tag}_summary.md")).read())


if __name__ == "__main__":
    main()
