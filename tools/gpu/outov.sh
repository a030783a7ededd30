timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_c1.json 2>gpurun_out/bench_c1.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_c1.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e'], d['ms_per_step'], d['roofline']['frac'])
P
