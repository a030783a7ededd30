#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_dist.py tests/test_gpu_algorithms.py -x -q -p no:cacheprovider > gpurun_out/r2ar_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ar_tests.log
for v in 0 1; do for cfg in C4 C3; do
if [ $v = 1 ]; then export FRPCA_OMEGA_PLACE_TILES=1; else unset FRPCA_OMEGA_PLACE_TILES; fi
timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/r2ar_prof_${cfg}_$v.json 2> gpurun_out/r2ar_prof_${cfg}_$v.err
done; done
