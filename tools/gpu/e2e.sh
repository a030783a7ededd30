for i in 1 2; do python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_e2e_$i.json 2> gpurun_out/bench_c1_e2e_$i.err; done
