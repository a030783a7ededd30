#!/bin/bash
# round 2: pipelined upload (values chunks -> first A*X), balanced panel plan, MLP gathers
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_tests.log
timeout 600 python tools/e2e_parts.py C3 > gpurun_out/r2g_e2eparts_c3.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 5 > gpurun_out/r2g_bench_c3.json 2> gpurun_out/r2g_bench_c3.err
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2g_launches_c3.csv python tools/run_csr_once.py C3 > gpurun_out/r2g_ncu.log 2>&1
