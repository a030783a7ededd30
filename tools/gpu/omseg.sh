#!/bin/bash
# A/B: Omega jump-ahead segment length (FRPCA_OMEGA_LOG2S)
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_algorithms.py -q -k "omega" > gpurun_out/omseg_tests.log 2>&1
timeout 900 python tools/ab_env.py --config C1 --runs 4 FRPCA_OMEGA_LOG2S=11 FRPCA_OMEGA_LOG2S=10 FRPCA_OMEGA_LOG2S=9 \
  > gpurun_out/omseg_C1.json 2> gpurun_out/omseg_C1.err
timeout 900 python tools/ab_env.py --config C4 --runs 3 FRPCA_OMEGA_LOG2S=12 FRPCA_OMEGA_LOG2S=11 FRPCA_OMEGA_LOG2S=13 \
  > gpurun_out/omseg_C4.json 2> gpurun_out/omseg_C4.err
