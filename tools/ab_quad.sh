# A/B of the quad dequeue (HS_QUAD) on C3, 64 RHS: device ms per application
for q in 0 1 0 1; do
  HS_QUAD=$q timeout 300 python tools/profile_cfg.py c3 --apps 3 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('HS_QUAD=$q', d['app_ms'])"
done
