#!/bin/bash
# Developer A/B of library variants (tools/build_variant.py) on one configuration:
#   bash tools/ab_variants.sh CFG VARIANT...   ("main" = the default build)
cfg=$1; shift
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="paper_2003_02585_b200/_variants/$v.so"; fi
  echo "== $v"
  HS_LIB_PATH=$lib python tools/profile_cfg.py $cfg --apps 3 2>&1 | tail -1
done
