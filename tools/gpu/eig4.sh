set -x
FRPCA_EIG=strict timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
FRPCA_EIG_TIMING=1 timeout 300 python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_eigc.json 2>gpurun_out/prof_C1_eigc.err
tail -5 gpurun_out/prof_C1_eigc.err
FRPCA_EIG=cusolver timeout 300 python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_eigd.json 2>gpurun_out/prof_C1_eigd.err
timeout 600 python bench.py > gpurun_out/bench_c1.json 2>gpurun_out/bench_c1.err; tail -c 1500 gpurun_out/bench_c1.json
