set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2a_gputest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2a_bench_c3.json 2> gpurun_out/r2a_bench_c3.err; echo "bench rc=$?"
cat gpurun_out/r2a_bench_c3.json
timeout 900 python bench.py --config C4 --no-cpu-baseline > gpurun_out/r2a_bench_c4.json 2> gpurun_out/r2a_bench_c4.err; echo "bench c4 rc=$?"
cat gpurun_out/r2a_bench_c4.json
