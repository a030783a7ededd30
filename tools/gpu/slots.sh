timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1 || exit 1
python tools/profile_run.py --config C4 --runs 3 > gpurun_out/prof_C4_alloc.json 2> gpurun_out/prof_C4_alloc.err
python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_nocpu.json 2> gpurun_out/bench_c1_nocpu.err
python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_cs.json 2>/dev/null
