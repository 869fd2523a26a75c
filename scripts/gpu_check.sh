# GPU tests + L2P diag + full bench (no CPU baseline)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/check.json 2>gpurun_out/check.err; echo bench rc=$?
python - <<'PY'
import json;d=json.load(open('gpurun_out/check.json'))
print('value',d['value'],'ms',d['ms_per_step'],'e2e_ms',d['e2e']['ms_per_step'])
print(d['stages_ms_per_step'])
for k,v in d['secondary'].items(): print(k, v.get('value'), v.get('ms_per_step'), v.get('stages_ms_per_step',{}).get('l2p'))
PY
