#!/bin/bash
cd "$(dirname "$0")/../.."
for c in C4 C3; do
timeout 900 python tools/e2e_ab.py $c 5 FRPCA_UPLOAD_PIPELINE=1 > gpurun_out/r2bb_lo_$c.json 2> gpurun_out/r2bb_lo_$c.err
FRPCA_BUILDER_PRIO=hi timeout 900 python tools/e2e_ab.py $c 5 FRPCA_UPLOAD_PIPELINE=1 > gpurun_out/r2bb_hi_$c.json 2> gpurun_out/r2bb_hi_$c.err
done
E2E_PER_CALL_PROFILE=1 FRPCA_DEBUG_TIMELINE=1 timeout 900 python tools/e2e_ab.py C4 1 FRPCA_UPLOAD_PIPELINE=1 > gpurun_out/r2bb_tl.json 2> gpurun_out/r2bb_tl.err
