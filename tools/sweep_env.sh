# Developer sweep of the solve engine's run-time knobs on one configuration (device ms per application):
#   bash tools/sweep_env.sh CFG [RHS] "VAR=val VAR2=val" ...
cfg=$1; rhs=$2; shift 2
for e in "$@"; do
  r=$(env $e timeout 300 python tools/profile_cfg.py $cfg --apps 2 --rhs $rhs 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(' '.join('%.2f' % x for x in d['app_ms']))")
  echo "[$e] $r"
done
