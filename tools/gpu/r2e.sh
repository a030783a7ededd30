#!/bin/bash
# round 2: per-kernel breakdowns (C4, C3, C2) at both register budgets
cd "$(dirname "$0")/../.."
for cfg in C4 C3 C2; do for mb in 4 2; do
FRPCA_SPMM_MINB=$mb timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/r2e_prof_${cfg}_minb$mb.json 2> gpurun_out/r2e_prof_${cfg}_minb$mb.err
done; done
