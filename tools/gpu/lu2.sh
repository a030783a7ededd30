timeout 600 python -m pytest tests -m gpu -q -x -k "lu or frpca" 2>&1 | tail -2
FRPCA_LU_TIMING=1 timeout 300 python tools/profile_run.py --config C1 --runs 2 > gpurun_out/prof_C1_lu.json 2>gpurun_out/prof_C1_lu.err
tail -4 gpurun_out/prof_C1_lu.err
python - <<'P'
import json
d=json.load(open('gpurun_out/prof_C1_lu.json'))
print({k:round(v['ms'],3) for k,v in d['kernels'].items() if 'lu' in k})
P
