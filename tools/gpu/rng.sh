timeout 600 python -m pytest tests/test_gpu_rng.py tests/test_gpu_algorithms.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
for c in C1 C4; do python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_rng.json 2>gpurun_out/prof_${c}_rng.err; done
