#!/bin/bash
# round 2: refresh the bench lines of C1, C2, C4 (C3 is the default workload)
cd "$(dirname "$0")/../.."
for c in C4 C2 C1; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/r2x_bench_$c.json 2> gpurun_out/r2x_bench_$c.err
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/r2x_bench_C1.err
