timeout 900 python -m pytest tests/test_gpu_validation.py -m gpu -q -x > gpurun_out/val_tests.log 2>&1
