# developer sweep: per-macro-step solve time vs split-K knobs (HS_KC / HS_KR / HS_SPLIT_DEPTH / HS_CRIT_GW)
for cfg in "8 4 8 8" "4 4 8 8" "2 4 8 8" "4 4 11 8" "8 8 8 8" "4 4 8 16" "2 4 11 8"; do
  set -- $cfg
  HS_KC=$1 HS_KR=$2 HS_SPLIT_DEPTH=$3 HS_CRIT_GW=$4 HS_STEP_TIMES=gpurun_out/st_$1_$2_$3_$4.csv HS_REPS=3 timeout 200 python tools/prof_step.py > /dev/null 2>&1
  echo "KC=$1 KR=$2 SD=$3 GW=$4 done"
done
