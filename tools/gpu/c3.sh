timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py tests/test_gpu_rng.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_nocpu.json 2> gpurun_out/bench_c1_nocpu.err
