#!/bin/bash
# Developer probe: C3 device ms per application, GPU tests, ncu launch list of the sweep kernels
timeout 300 python tools/profile_cfg.py c3 --apps 4 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('app_ms', d['app_ms'])"
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"accumulate_all|inject|extract|rhs_init|nonzero|residual|transpose|reduce" --log-file gpurun_out/sweepk_launches.csv \
  python tools/profile_cfg.py c3 --apps 1 > gpurun_out/sweepk_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open('gpurun_out/sweepk_launches.csv') if l.startswith('"')))
h = rows[0]; ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
idi = h.index('ID')
d = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter()
for r in rows[1:]:
    k = r[ki].split('(')[0].split('::')[-1]
    d[k][r[mi]] += float(r[vi].replace(',', ''))
    if r[mi] == 'gpu__time_duration.sum': cnt[k] += 1
for k, m in sorted(d.items(), key=lambda kv: -kv[1]['gpu__time_duration.sum']):
    t = m['gpu__time_duration.sum']  # ns
    by = m['dram__bytes_read.sum'] + m['dram__bytes_write.sum']
    print(f"{k:40s} n={cnt[k]:5d} total {t/1e6:8.2f} ms  {t/1e3/cnt[k]:8.1f} us/launch  {by/t:7.0f} GB/s")
PY
