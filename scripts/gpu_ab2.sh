# GPU tests, then the headline bench (+ secondary unless NOSEC) for VAR=0 and VAR=1
VAR=${1:-FC2T2_M2L_DENSE}
timeout 1200 python -m pytest tests -m gpu -q -x ${TESTK:+-k "$TESTK"} 2>&1 | tail -4
for v in 0 1; do
  echo "== $VAR=$v"
  env $VAR=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${NOSEC:+--no-secondary} > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err || tail -5 gpurun_out/ab_$v.err
  python - <<PY
import json;d=json.load(open('gpurun_out/ab_$v.json'))
print('value',round(d['value']/1e9,3),'G ms',round(d['ms_per_step'],3),'e2e_ms',round(d['e2e']['ms_per_step'],3))
print({k:v for k,v in d['stages_ms_per_step'].items()})
for k,s in d.get('secondary',{}).items(): print(k, s.get('value'), s.get('ms_per_step'))
PY
done
