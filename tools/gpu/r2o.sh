#!/bin/bash
# round 2: fused Omega (generation + polar in one pass, row-major placement)
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_tests.log
for cfg in C4 C1 C3; do
timeout 600 python tools/profile_run.py --config $cfg --runs 3 > gpurun_out/r2o_prof_$cfg.json 2> gpurun_out/r2o_prof_$cfg.err
done
