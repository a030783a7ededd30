timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_emit|k_gen" -c 2 -o gpurun_out/rng -f python tools/profile_run.py --config C1 --runs 1 > gpurun_out/ncu_rng.log 2>&1
tail -1 gpurun_out/ncu_rng.log
