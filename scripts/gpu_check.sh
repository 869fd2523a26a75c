# GPU tests + L2P diag + full bench (no CPU baseline)
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
LEVEL=5 RHO=4 M=10000000 timeout 300 python scripts/diag_l2p.py 2>&1 | tail -2
LEVEL=6 RHO=6 timeout 300 python scripts/diag_l2p.py 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/check.json 2>gpurun_out/check.err; echo bench rc=$?
python - <<'PY'
import json;d=json.load(open('gpurun_out/check.json'))
print('value',d['value'],'ms',d['ms_per_step'],'e2e_ms',d['e2e']['ms_per_step'])
print(d['stages_ms_per_step'])
for k,v in d['secondary'].items(): print(k, v.get('value'), v.get('ms_per_step'), v.get('stages_ms_per_step',{}).get('l2p'))
PY
