for m in 3 14 22; do HS_TRACE=gpurun_out/trace_m$m.csv HS_TRACE_STEP=$m HS_REPS=2 timeout 300 python tools/prof_step.py > gpurun_out/trace_m$m.log 2>&1; done
ls -la gpurun_out
