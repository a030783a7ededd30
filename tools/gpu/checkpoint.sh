# round checkpoint: tests, bench (both arms), launch list, SpMM full capture
set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --impl reference > gpurun_out/bench_c1_ref.json 2> gpurun_out/bench_c1_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/profile_run.py --config C1 --runs 1 > gpurun_out/prof_c1_once.json 2>/dev/null && \
  ncu --set full --clock-control none --import-source on --kernel-name regex:"k_spmm|k_combine" -c 12 \
      -o gpurun_out/c1_spmm -f python tools/profile_run.py --config C1 --runs 1 > gpurun_out/ncu_full.log 2>&1
