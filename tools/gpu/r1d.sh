#!/bin/bash
cd "$(dirname "$0")/../.."
for cfg in C1 C4 C3; do
  timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/cb_${cfg}_cs.json 2> /dev/null
  FRPCA_COMBINE_LDG=1 timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/cb_${cfg}_ldg.json 2> /dev/null
  FRPCA_COMBINE1=1 timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/cb_${cfg}_old.json 2> /dev/null
  FRPCA_DEBUG_PANELS=1 timeout 600 python tools/profile_run.py --config $cfg --runs 1 2>&1 >/dev/null | grep panels > gpurun_out/cb_${cfg}_plan.txt
done
