#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "spmm" > gpurun_out/r2aj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2aj_tests.log
for cfg in C3 C4 C2 C1; do
timeout 900 python tools/ab_env.py --config $cfg --runs 3 FRPCA_AX_SLAB=256 FRPCA_AX_SLAB=100 FRPCA_AX_SLAB=64 > gpurun_out/r2aj_ab_$cfg.json 2> gpurun_out/r2aj_ab_$cfg.err
done
