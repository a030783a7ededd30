timeout 600 python -m pytest tests -m gpu -q -x -k "rng or omega or gaussian or sketch or frpca" 2>&1 | tail -2
timeout 300 python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_rng.json 2>gpurun_out/prof_C1_rng.err
python - <<'P'
import json
d=json.load(open('gpurun_out/prof_C1_rng.json'))
print({k:round(v['ms'],3) for k,v in d['kernels'].items() if 'omega' in k})
P
