timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python scripts/diag_step.py > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -o gpurun_out/step_q python scripts/diag_step.py > /dev/null 2>&1; python scripts/ncu_traffic.py gpurun_out/step_q.ncu-rep 1 gpurun_out/traffic_q.json > /dev/null 2>&1
python - <<'PY'
import json; d=json.load(open('gpurun_out/traffic_q.json'))
print({k: round(v*1000,1) for k,v in sorted(d['serial_ms_per_step'].items(), key=lambda kv:-kv[1])}, round(sum(d['serial_ms_per_step'].values()),4))
PY
timeout 600 python bench.py --no-cpu-baseline --no-secondary > gpurun_out/q.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/q.json'));print(d['ms_per_step'], d['e2e']['ms_per_step'], d['graphed']['ms_per_step'])"
