# developer comparison of library variants (paper_2003_02585_b200/_variants/*.so, tools/build_variant.py)
for v in base "$@"; do
  if [ "$v" = base ]; then unset HS_LIB_PATH; else export HS_LIB_PATH=paper_2003_02585_b200/_variants/$v.so; fi
  HS_STEP_TIMES=gpurun_out/var_$v.csv HS_REPS=3 timeout 200 python tools/prof_step.py 2>&1 | grep "app 2" | cut -c1-60
done
