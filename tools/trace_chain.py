"""Developer tool: critical chain of one solve pass from an HS_TRACE csv (per-item timestamps).
Walks back from the last-finishing item: a front's predecessor is the front of the same task
(pass 0: a child, pass 1: the parent) whose last item finished latest before the front's first
ready time. Usage: python tools/trace_chain.py trace.csv"""
import sys
import pandas as pd

d = pd.read_csv(sys.argv[1])
d = d[(d.t_deq > 0) & (d.t_done > 0)].copy()
T0 = d.t_deq.min()
for c in ["t_deq", "t_ready", "t_loop", "t_red", "t_done"]:
    d[c] = (d[c] - T0) / 1e3
for p in [0, 1]:
    e = d[d["pass"] == p]
    last = e.loc[e.t_done.idxmax()]
    es = e[e["sub"] == last["sub"]]
    g = es.groupby("front").agg(k=("k", "first"), m=("m", "first"), n=("idx", "size"), deq0=("t_deq", "min"),
                                deq1=("t_deq", "max"), rdy0=("t_ready", "min"), rdy1=("t_ready", "max"),
                                loop=("t_loop", "max"), done=("t_done", "max"), ns=("nsteps", "max"))
    f = int(last["front"])
    chain = []
    while True:
        row = g.loc[f]
        chain.append((f, row))
        cand = g[(g.done <= row.rdy0 + 0.05) & (g.index != f)]
        if cand.empty:
            break
        f = int(cand.done.idxmax())
    print(f"pass {p}: span {e.t_done.max() - e.t_deq.min():.1f} us, sub {last['sub']}, chain of {len(chain)} fronts")
    print(f"{'front':>6} {'k':>4} {'m':>4} {'n':>3} {'deq0':>6} {'deq1':>6} {'rdy0':>6} {'rdy1':>6} {'loop':>6} {'done':>6} {'ns':>3} {'level_us':>8}")
    prev = None
    for f, r in reversed(chain):
        lv = r.done - (prev if prev is not None else r.rdy0)
        print(f"{f:6d} {int(r.k):4d} {int(r.m):4d} {int(r.n):3d} {r.deq0:6.1f} {r.deq1:6.1f} {r.rdy0:6.1f} {r.rdy1:6.1f} {r.loop:6.1f} {r.done:6.1f} {int(r.ns):3d} {lv:8.1f}")
        prev = r.done
