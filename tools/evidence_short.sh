set -x
# the evidence job without the sweep-kernel full capture (tools/evidence_job.sh is the whole run)
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/r2_gputests.log 2>&1; tail -3 gpurun_out/r2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
timeout 400 python tools/check_c5.py > gpurun_out/r2_c5.log 2>&1; tail -1 gpurun_out/r2_c5.log | cut -c1-400
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.log 2>&1; tail -c 600 gpurun_out/r2_bench.log
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c2.log 2>&1; tail -c 300 gpurun_out/r2_bench_c2.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_bench.log 2>&1; wc -l gpurun_out/r2_launches.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve6 -s 70 -c 2 -o gpurun_out/r2_solve_full python tools/profile_cfg.py c3 --apps 1 > gpurun_out/r2_ncu_full.log 2>&1; tail -2 gpurun_out/r2_ncu_full.log
