timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sytrd -c 1 -o gpurun_out/sytrd -f python tools/profile_run.py --config C1 --runs 1 > gpurun_out/ncu_sytrd.log 2>&1
tail -3 gpurun_out/ncu_sytrd.log
