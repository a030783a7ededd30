export FRPCA_DEBUG_PANELS=1
for c in C1 C4 C3; do python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_p32.json 2>gpurun_out/prof_${c}_p32.err; done
