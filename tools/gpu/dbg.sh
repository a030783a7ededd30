timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "panel" > gpurun_out/dbg1.log 2>&1
timeout 600 python -m pytest tests/test_gpu_algorithms.py -m gpu -q -k "panelled" > gpurun_out/dbg2.log 2>&1
FRPCA_LU_GLOBAL=1 timeout 600 python -m pytest tests/test_gpu_algorithms.py -m gpu -q -k "panelled" > gpurun_out/dbg3.log 2>&1
