#!/bin/bash
cd "$(dirname "$0")/../.."
# the builder context (and its stream) is created once per process: one process per variant
timeout 900 python tools/e2e_ab.py C3 10 FRPCA_UPLOAD_PIPELINE=1 > gpurun_out/r2aw_hi.json 2> gpurun_out/r2aw_hi.err
FRPCA_BUILDER_PRIO=lo timeout 900 python tools/e2e_ab.py C3 10 FRPCA_UPLOAD_PIPELINE=1 > gpurun_out/r2aw_lo.json 2> gpurun_out/r2aw_lo.err
FRPCA_BUILDER_PRIO=lo E2E_PER_CALL_PROFILE=1 FRPCA_DEBUG_TIMELINE=1 timeout 900 python tools/e2e_ab.py C3 2 FRPCA_UPLOAD_PIPELINE=1 > gpurun_out/r2aw_lo_tl.json 2> gpurun_out/r2aw_lo_tl.err
