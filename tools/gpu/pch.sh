export FRPCA_DEBUG_PANELS=1
for pc in 64 128 256 1024; do for c in C1 C4; do FRPCA_PANEL_CHUNK=$pc python tools/profile_run.py --config $c --runs 2 > gpurun_out/prof_${c}_pc$pc.json 2>/dev/null; done; done
