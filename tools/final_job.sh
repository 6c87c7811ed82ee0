# the round's closing run: GPU tests, smoke, the C3 and C2 bench lines (ncu artefacts come from evidence_job.sh)
set -x
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/r2_gputests.log 2>&1; tail -3 gpurun_out/r2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.log 2>&1; tail -c 400 gpurun_out/r2_bench.log
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c2.log 2>&1; tail -c 300 gpurun_out/r2_bench_c2.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1; tail -c 400 gpurun_out/r2_bench_ref.log
