#!/bin/bash
# combine2 / LU-threads checks and timings
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "combine2 or lu or spmm" > gpurun_out/t_r1c.log 2>&1
FRPCA_LU_SMEM_THREADS=1024 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "lu" > gpurun_out/t_r1c_lu1024.log 2>&1
for cfg in C1 C4; do
  timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/c2_${cfg}_new.json 2> /dev/null
  FRPCA_COMBINE1=1 timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/c2_${cfg}_old.json 2> /dev/null
done
FRPCA_LU_SMEM_THREADS=1024 timeout 300 python tools/profile_run.py --config C1 --runs 3 > gpurun_out/lu1024_C1.json 2> /dev/null
FRPCA_LU_TIMING=1 timeout 600 python tools/profile_run.py --config C2 --runs 2 > /dev/null 2> gpurun_out/lutiming_C2.err
