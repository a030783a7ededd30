#!/bin/bash
# A*X L1/L2-hint sweep: per-kernel event breakdown per config and FRPCA_HINT_MB
cd "$(dirname "$0")/../.."
for cfg in ${CFGS:-C1 C2 C3 C4}; do
  for mb in ${MBS:-0 64 128}; do
    FRPCA_HINT_MB=$mb timeout 600 python tools/profile_run.py --config $cfg --runs 3 \
      > gpurun_out/hint${TAG}_${cfg}_${mb}.json 2> gpurun_out/hint${TAG}_${cfg}_${mb}.err
  done
done
