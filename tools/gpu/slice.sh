FRPCA_SPMM_SLICE=128 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py -m gpu -q -x > gpurun_out/gpu_tests128.log 2>&1
for sw in 128; do for c in C1 C2 C3 C4; do FRPCA_SPMM_SLICE=$sw python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_sw$sw.json 2>/dev/null; done; done
for c in C1 C2 C3 C4; do python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_sw256.json 2>/dev/null; done
