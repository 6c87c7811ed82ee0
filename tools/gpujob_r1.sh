# Round-1 evidence job (run under gpurun): parity, smoke, bench, ncu launch list, ncu full capture.
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; tail -c 3000 gpurun_out/bench_r1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r1.log 2>&1
HS_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve6 --launch-skip 28 --launch-count 2 -o gpurun_out/solve_full_r1 python tools/prof_step.py > gpurun_out/ncu_full_r1.log 2>&1
HS_REPS=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:solve6 --csv --log-file gpurun_out/solve_dram_all.csv python tools/prof_step.py > gpurun_out/solve_dram_all.log 2>&1
ls -la gpurun_out | tail -8
timeout 900 python tools/check_c5.py > gpurun_out/c5.log 2>&1; tail -c 600 gpurun_out/c5.log
timeout 900 python tools/run_config.py c3 --ref-full > gpurun_out/c3.log 2>&1; tail -c 600 gpurun_out/c3.log
