#!/bin/bash
# round checkpoint: tests, smoke, bench (both arms), other configs, launch list, SpMM ncu capture
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_c1_ref.json 2> gpurun_out/bench_c1_ref.err
for c in C2 C3 C4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_short.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmm" -c 6 -o gpurun_out/spmm_c1 -f \
  python tools/profile_run.py --config C1 --runs 1 > gpurun_out/ncu_spmm.log 2>&1
