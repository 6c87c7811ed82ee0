"""Developer tool: from an HS_TRACE csv, warp occupancy over time (busy / in k-loop / waiting for
readiness) and, per front-size class, the warp time inside and outside the k-loop.
Usage: python tools/trace_classes.py trace.csv"""
import sys
import numpy as np
import pandas as pd

d = pd.read_csv(sys.argv[1])
d = d[(d.t_deq > 0) & (d.t_done > 0)].copy()
for p in (0, 1):
    e = d[d["pass"] == p]
    T0, T1 = e.t_deq.min(), e.t_done.max()
    nb = 16
    edges = np.linspace(T0, T1, nb + 1)
    print(f"pass {p}: span {(T1 - T0) / 1e3:.1f} us, {len(e)} items")

    def occ(a, b):
        return [np.clip(np.minimum(b, edges[i + 1]).astype(float) - np.maximum(a, edges[i]).astype(float), 0, None).sum()
                / (edges[i + 1] - edges[i]) for i in range(nb)]
    for name, a, b in (("busy", e.t_deq, e.t_done), ("loop", e.t_ready, e.t_loop), ("ready", e.t_deq, e.t_ready)):
        print(f"  {name:6s}", " ".join(f"{x:5.0f}" for x in occ(a.values, b.values)))
    e = e.assign(rdy=(e.t_ready - e.t_deq) / 1e3, lt=(e.t_loop - e.t_ready) / 1e3, post=(e.t_done - e.t_loop) / 1e3)
    g = e.groupby(pd.cut(e.k, [0, 8, 16, 32, 48, 64, 128, 300]), observed=True).agg(
        items=("lt", "size"), ready_us=("rdy", "sum"), loop_us=("lt", "sum"), post_us=("post", "sum"), ksteps=("nsteps", "sum"))
    g["us_per_kstep"] = g.loop_us / g.ksteps
    g["post_per_item"] = g.post_us / g["items"]
    print(g.round(2).to_string())
