# round 2: dist fix + bitwise Omega tests, then e2e diagnosis at C3
set -x
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_rng.py tests/test_gpu_algorithms.py -x -q -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2b_tests.log
timeout 600 python tools/e2e_parts.py C3 > gpurun_out/r2b_e2eparts_c3.txt 2>&1; echo "parts rc=$?"
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 8 > gpurun_out/r2b_bench_c3.json 2> gpurun_out/r2b_bench_c3.err; echo "bench rc=$?"
free -g; nproc; nvidia-smi --query-gpu=memory.used,memory.total --format=csv
