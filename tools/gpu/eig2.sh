FRPCA_EIG_TIMING=1 python tools/profile_run.py --config C1 --runs 1 > gpurun_out/prof_C1_eig.json 2>gpurun_out/prof_C1_eig.err
