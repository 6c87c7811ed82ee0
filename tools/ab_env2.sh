#!/bin/bash
# Developer A/B: C3 device ms per application under environment switches. usage: tools/ab_env2.sh "A=1" "B=2 C=3" ...
for e in "" "$@"; do
  echo "== env: $e"
  env $e timeout 300 python tools/profile_cfg.py c3 --apps 4 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('app_ms', [round(x,2) for x in d['app_ms']], 'solve_s', round(d['profile']['solve_seconds'],4))"
done
