#!/bin/bash
# round 2: launch list of one warm e2e call (frpca_run_csr) at C3
cd "$(dirname "$0")/../.."
timeout 600 python tools/run_csr_once.py C3 > gpurun_out/r2f_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2f_launches_c3.csv python tools/run_csr_once.py C3 > gpurun_out/r2f_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_ncu.log
