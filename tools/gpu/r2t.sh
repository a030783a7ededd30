#!/bin/bash
# round 2: ncu full capture of C3's SpMM / dense / Omega kernels + launch list of the C3 bench step
cd "$(dirname "$0")/../.."
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm|k_gram4|k_gemm_tma|k_gen_polar|k_place|k_combine" -c 14 \
   -o gpurun_out/r2t_c3_full -f python tools/profile_run.py --config C3 --runs 1 > gpurun_out/r2t_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_ncu_full.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2t_bench_short.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_launches_c3.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2t_ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_ncu_launch.log
