"""Developer tool: key metrics of every kernel in an .ncu-rep (ncu --page details --csv)."""
import csv, io, subprocess, sys
KEYS = ["Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Eligible Warps Per Scheduler", "No Eligible"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
for i in sorted(set(r["ID"] for r in rows), key=int):
    rs = [r for r in rows if r["ID"] == i]
    print("==", i, rs[0]["Kernel Name"][:70])
    for r in rs:
        if r["Metric Name"] in KEYS:
            print(f"   {r['Metric Name']:40s} {r['Metric Unit']:12s} {r['Metric Value']}")
