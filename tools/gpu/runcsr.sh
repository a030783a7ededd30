timeout 900 python -m pytest tests/test_gpu_algorithms.py -m gpu -q -x -k "run_csr" > gpurun_out/runcsr_tests.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_nocpu.json 2> gpurun_out/bench_c1_nocpu.err
python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
