#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_dist.py tests/test_gpu_algorithms.py -x -q -p no:cacheprovider > gpurun_out/r2y_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_tests.log
FRPCA_DEBUG_ALLOC=1 timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/r2y_bench_C4.json 2> gpurun_out/r2y_bench_C4.err
timeout 600 python tools/profile_run.py --config C4 --runs 3 > gpurun_out/r2y_prof_C4.json 2> gpurun_out/r2y_prof_C4.err
