#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_rng.py tests/test_gpu_dist.py -x -q -p no:cacheprovider -k "stream or window or omega or segment" > gpurun_out/r2bn_tests.log 2>&1
FRPCA_OMEGA_ROUND=8 timeout 600 python -m pytest tests/test_gpu_rng.py tests/test_gpu_dist.py tests/test_gpu_algorithms.py -x -q -p no:cacheprovider -k "stream or window or omega or segment" >> gpurun_out/r2bn_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bn_tests.log
for v in 4 8; do for cfg in C4 C1; do
FRPCA_OMEGA_ROUND=$v timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/r2bn_prof_${cfg}_$v.json 2> gpurun_out/r2bn_prof_${cfg}_$v.err
done; done
