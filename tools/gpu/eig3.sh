set -x
FRPCA_EIG=strict timeout 600 python -m pytest tests -m gpu -x -q -k "eig or frpca" 2>&1 | tail -15
FRPCA_EIG=custom FRPCA_EIG_TIMING=1 timeout 300 python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_eigc.json 2>gpurun_out/prof_C1_eigc.err
tail -5 gpurun_out/prof_C1_eigc.err
timeout 300 python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_eigd.json 2>gpurun_out/prof_C1_eigd.err
