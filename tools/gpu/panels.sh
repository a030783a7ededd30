timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
for c in C1 C4 C3 C2; do python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_p32.json 2>gpurun_out/prof_${c}_p32.err; done
for mb in 16 64; do for c in C1 C4; do FRPCA_PANEL_MB=$mb python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_p$mb.json 2>/dev/null; done; done
FRPCA_NO_PANELS=1 python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_nop.json 2>/dev/null
