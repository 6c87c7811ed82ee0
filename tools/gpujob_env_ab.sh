# developer A/B of environment knobs: each argument is one "VAR=val VAR2=val" setting ("-" = none)
for rep in 1 2; do
for cfg in "$@"; do
  if [ "$cfg" = "-" ]; then e=""; else e="$cfg"; fi
  echo -n "[$cfg] "; env $e HS_REPS=3 timeout 200 python tools/prof_step.py 2>&1 | grep "app 2" | cut -c1-70
done
done
