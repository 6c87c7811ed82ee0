"""Developer tool: where a solve launch's warp time goes, from an HS_TRACE csv (per-item
timestamps: dequeue, ready (dependencies + index staging), k-loop done, split-K reduced, done).
Sums each phase over all items of each pass and prints the share of the warp-time total.
Usage: python tools/item_phases.py trace.csv"""
import sys
import pandas as pd

d = pd.read_csv(sys.argv[1])
d = d[(d.t_deq > 0)].copy()
for p in (0, 1):
    e = d[d["pass"] == p]
    live = e[e.t_done > 0]
    skipped = len(e) - len(live)
    ph = {"ready (records, deps, index)": (live.t_ready - live.t_deq).sum(),
          "k-loop": (live.t_loop - live.t_ready).sum(),
          "split-K reduce": (live.t_red - live.t_loop).clip(lower=0).sum(),
          "finalize + signal": (live.t_done - live.t_red).clip(lower=0).sum()}
    tot = sum(ph.values())
    span = (live.t_done.max() - e.t_deq.min()) / 1e3
    print(f"pass {p}: {len(e)} items ({skipped} skipped at run time), span {span:.1f} us, "
          f"k-steps {live.nsteps.sum()}, mean k-steps per item {live.nsteps.mean():.1f}")
    for k, v in ph.items():
        print(f"   {k:32s} {100 * v / tot:5.1f}%   mean {v / max(len(live), 1) / 1e3:6.2f} us")
