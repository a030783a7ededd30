#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_dist.py tests/test_gpu_algorithms.py -x -q -p no:cacheprovider > gpurun_out/r2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.log
for cfg in C4 C1 C3 C2; do
timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/r2s_prof_$cfg.json 2> gpurun_out/r2s_prof_$cfg.err
done
