#!/bin/bash
# A/B: A^T*Y cold rows concurrent with the panel chunks (FRPCA_COLD_CONCURRENT),
# SpMM items from a global counter (FRPCA_SPMM_DYNAMIC)
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "cold_concurrent or panelled or dynamic" > gpurun_out/cold_tests.log 2>&1
for c in C1 C2 C4 C3; do
  timeout 900 python tools/ab_env.py --config $c --runs 5 FRPCA_SPMM_DYNAMIC=0 FRPCA_SPMM_DYNAMIC=2 FRPCA_SPMM_DYNAMIC=1 \
    FRPCA_COLD_CONCURRENT=1,FRPCA_SPMM_DYNAMIC=2 FRPCA_COLD_CONCURRENT=1,FRPCA_SPMM_DYNAMIC=1 \
    > gpurun_out/cold_$c.json 2> gpurun_out/cold_$c.err
done
