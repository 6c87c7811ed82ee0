# developer sweep of runtime knobs (HS_SPLIT_DEPTH / HS_KC / HS_KR)
for cfg in "8 8 4" "6 8 4" "10 8 4" "8 4 4" "8 8 8" "8 16 4"; do
  set -- $cfg
  echo -n "SD=$1 KC=$2 KR=$3: "; HS_SPLIT_DEPTH=$1 HS_KC=$2 HS_KR=$3 HS_REPS=3 timeout 100 python tools/prof_step.py 2>&1 | grep "app 2" | cut -c1-105
done
