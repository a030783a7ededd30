#!/bin/bash
# parity variants at C1, GEMM warp sweep
cd "$(dirname "$0")/../.."
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm_warps or l2_hints or eig_svd" > gpurun_out/t_r1b.log 2>&1
timeout 600 python tools/parity_variants.py --config C1 --out gpurun_out/pvar_C1.json > gpurun_out/pvar_C1.log 2>&1
for cfg in C1 C3; do
  for w in 8 16; do
    FRPCA_GEMM_WARPS=$w timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/gw_${cfg}_${w}.json 2> gpurun_out/gw_${cfg}_${w}.err
  done
done
