#!/bin/bash
# host-side id narrowing at upload: tests, e2e A/B at C3 and C4, timeline
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nproc > gpurun_out/n_nproc.txt; lscpu | head -20 >> gpurun_out/n_nproc.txt
timeout 900 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_load.py -x -q -p no:cacheprovider > gpurun_out/n_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n_tests.log
timeout 900 python tools/e2e_ab.py C3 6 FRPCA_HOST_NARROW=0 FRPCA_HOST_NARROW=1 > gpurun_out/n_ab_c3.json 2> gpurun_out/n_ab_c3.err
FRPCA_DEBUG_TIMELINE=1 timeout 600 python tools/e2e_ab.py C3 1 FRPCA_HOST_NARROW=1 > gpurun_out/n_tl_c3.json 2> gpurun_out/n_tl_c3.err
timeout 900 python tools/e2e_ab.py C4 4 FRPCA_HOST_NARROW=0 FRPCA_HOST_NARROW=1 > gpurun_out/n_ab_c4.json 2> gpurun_out/n_ab_c4.err
