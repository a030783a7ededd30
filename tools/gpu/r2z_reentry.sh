#!/bin/bash
# re-entry check after a container rebuild: whole GPU suite, smoke, default bench
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/z_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/z_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/z_smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
