#!/bin/bash
cd "$(dirname "$0")/../.."
for cfg in C4 C1 C2; do
timeout 900 python tools/ab_env.py --config $cfg --runs 4 FRPCA_COLD_CONCURRENT=1 FRPCA_COLD_CONCURRENT=0 > gpurun_out/r2ai_ab_$cfg.json 2> gpurun_out/r2ai_ab_$cfg.err
done
