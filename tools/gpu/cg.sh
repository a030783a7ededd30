#!/bin/bash
# A/B: L1-bypassing gathers (FRPCA_GATHER_CG); panel size with dynamic items
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "gather_cg or dynamic or cold" > gpurun_out/cg_tests.log 2>&1
for c in C1 C2 C4 C3; do
  timeout 900 python tools/ab_env.py --config $c --runs 4 FRPCA_GATHER_CG=0 FRPCA_GATHER_CG=1 \
    > gpurun_out/cg_$c.json 2> gpurun_out/cg_$c.err
done
for c in C1 C3; do
  timeout 900 python tools/ab_env.py --config $c --runs 4 --reupload FRPCA_PANEL_MB=32 FRPCA_PANEL_MB=16 FRPCA_PANEL_MB=64 \
    > gpurun_out/pmb_$c.json 2> gpurun_out/pmb_$c.err
done
