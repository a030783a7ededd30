timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
for c in C1 C4; do python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_gm.json 2>/dev/null; done
