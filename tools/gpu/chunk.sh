#!/bin/bash
# A/B: work-list chunk size (items per warp) with dynamic item scheduling
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py -q -x > gpurun_out/chunk_tests.log 2>&1
for c in C1 C2 C4 C3; do
  timeout 900 python tools/ab_env.py --config $c --runs 4 --reupload FRPCA_CHUNK_ITEMS=16 FRPCA_CHUNK_ITEMS=32 FRPCA_CHUNK_ITEMS=64 \
    > gpurun_out/chunk_$c.json 2> gpurun_out/chunk_$c.err
done
