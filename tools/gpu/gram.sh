timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "gram or eig_svd" > gpurun_out/gram_tests.log 2>&1
for c in C1 C4; do python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_g3.json 2>/dev/null; done
