#!/bin/bash
# round 2 checkpoint: full GPU suite, smoke, bench (both arms), launch list
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/ck_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ck_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ck_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ck_smoke.log
timeout 900 python bench.py > gpurun_out/ck_bench_c3.json 2> gpurun_out/ck_bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/ck_bench_c3_ref.json 2> gpurun_out/ck_bench_c3_ref.err
