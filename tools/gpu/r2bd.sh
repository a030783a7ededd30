#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/r2bd_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bd_tests.log
for c in C3 C1 C2 C4; do
timeout 1200 python tools/ab_env.py --config $c --runs 4 --reupload FRPCA_ITEM_ORDER=0 FRPCA_ITEM_ORDER=1 > gpurun_out/r2bd_ab_$c.json 2> gpurun_out/r2bd_ab_$c.err
done
