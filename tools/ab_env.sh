#!/bin/bash
# Developer A/B of environment switches on one configuration:
#   bash tools/ab_env.sh CFG "ENV=.. ENV2=.." "..."   ("-" = no switches)
cfg=$1; shift
for e in "$@"; do
  echo "== $e"
  if [ "$e" = - ]; then e=""; fi
  env $e python tools/profile_cfg.py $cfg --apps 3 2>&1 | tail -1
done
