timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "eig" > gpurun_out/eig_tests.log 2>&1
FRPCA_EIG_TIMING=1 python tools/profile_run.py --config C1 --runs 1 > gpurun_out/prof_C1_eig.json 2>gpurun_out/prof_C1_eig.err
