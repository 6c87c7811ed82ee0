for v in f3b4 f2b4 f2b3 f4b4 f2b2 f3b4; do
  echo -n "$v: "; HS_LIB_PATH=paper_2003_02585_b200/_variants/$v.so HS_REPS=3 HS_STEP_TIMES=gpurun_out/st_$v.csv timeout 100 python tools/prof_step.py 2>&1 | grep "app 2" | cut -c1-110
done
