#!/bin/bash
# round 2: register-budget and shared-memory hot-row A/B for the gather kernels
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "hot_rows_in_smem or register_budget" > gpurun_out/r2d_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_tests.log
for cfg in C3 C1 C2 C4; do
timeout 900 python tools/ab_env.py --config $cfg --runs 4 FRPCA_SPMM_MINB=4 FRPCA_SPMM_MINB=2 FRPCA_SPMM_MINB=1 \
  FRPCA_SPMM_HS=1,FRPCA_SPMM_HS_THREADS=512 FRPCA_SPMM_HS=1,FRPCA_SPMM_HS_THREADS=512,FRPCA_SPMM_MINB=2 \
  FRPCA_SPMM_HS=1,FRPCA_SPMM_HS_THREADS=1024 > gpurun_out/r2d_ab_$cfg.json 2> gpurun_out/r2d_ab_$cfg.err
done
