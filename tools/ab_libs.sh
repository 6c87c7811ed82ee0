#!/bin/bash
# Developer A/B: C3 device ms per application for library variants (HS_LIB_PATH), plus the ncu time /
# DRAM GB/s of the kernels matching $KREGEX.  usage: tools/ab_libs.sh main base acc2 ...
KREGEX=${KREGEX:-accumulate_all}
for v in "$@"; do
  if [ "$v" = main ]; then unset HS_LIB_PATH; else export HS_LIB_PATH=$PWD/paper_2003_02585_b200/_variants/$v.so; fi
  echo "== $v"
  timeout 300 python tools/profile_cfg.py c3 --apps 4 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('app_ms', [round(x,2) for x in d['app_ms']])"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"$KREGEX" --log-file gpurun_out/ab_$v.csv python tools/profile_cfg.py c3 --apps 1 > gpurun_out/ab_$v.log 2>&1
  python - gpurun_out/ab_$v.csv <<'PY'
import csv, collections, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]; ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
d = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter()
for r in rows[1:]:
    k = r[ki].split('(')[0].split('::')[-1]
    d[k][r[mi]] += float(r[vi].replace(',', ''))
    if r[mi] == 'gpu__time_duration.sum': cnt[k] += 1
for k, m in sorted(d.items(), key=lambda kv: -kv[1]['gpu__time_duration.sum']):
    t = m['gpu__time_duration.sum']; by = m['dram__bytes_read.sum'] + m['dram__bytes_write.sum']
    print(f"  {k:36s} n={cnt[k]:5d} total {t/1e6:8.2f} ms  {t/1e3/cnt[k]:8.1f} us/launch  {by/t:7.0f} GB/s")
PY
done
