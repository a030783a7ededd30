#!/bin/bash
# round 2 re-entry: full GPU suite on the restored tree, then the C3 bench
cd "$(dirname "$0")/../.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2c_smi.txt
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c_smoke.log
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/r2c_bench_c3.json 2> gpurun_out/r2c_bench_c3.err; echo "bench rc=$?" >> gpurun_out/r2c_bench_c3.err
