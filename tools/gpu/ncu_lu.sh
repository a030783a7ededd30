timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lu_smem -c 1 -o gpurun_out/lu -f python tools/profile_run.py --config C1 --runs 1 > gpurun_out/ncu_lu.log 2>&1
tail -2 gpurun_out/ncu_lu.log
