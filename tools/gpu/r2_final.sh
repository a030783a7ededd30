#!/bin/bash
# round 2 final evidence: bench lines C3 (default, both arms' shape) + C1/C2/C4, ncu of C3's kernels, launch list
cd "$(dirname "$0")/../.."
timeout 900 python bench.py > gpurun_out/fin_bench_c3.json 2> gpurun_out/fin_bench_c3.err
for c in C4 C2 C1; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/fin_bench_$c.json 2> gpurun_out/fin_bench_$c.err
done
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm|k_gram4|k_gemm_tma|k_combine" -c 12 \
   -o gpurun_out/fin_c3_full -f python tools/profile_run.py --config C3 --runs 1 > gpurun_out/fin_ncu_full.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin_bench_short.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c3.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin_ncu_launch.log 2>&1
