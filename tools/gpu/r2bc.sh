#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_algorithms.py -x -q -p no:cacheprovider -k "run_csr" > gpurun_out/r2bc_tests.log 2>&1
FRPCA_SORT_ON_BUILDER=1 timeout 600 python -m pytest tests/test_gpu_algorithms.py -x -q -p no:cacheprovider -k "run_csr" >> gpurun_out/r2bc_tests.log 2>&1; echo rc=$? >> gpurun_out/r2bc_tests.log
for c in C3 C4; do
timeout 900 python tools/e2e_ab.py $c 5 FRPCA_SORT_ON_BUILDER=0 FRPCA_SORT_ON_BUILDER=1 > gpurun_out/r2bc_$c.json 2> gpurun_out/r2bc_$c.err
done
