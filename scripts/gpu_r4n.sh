mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_expansion.py -q -x  2>&1 | tail -3
timeout 300 python scripts/diag_timeline.py > gpurun_out/r4n_timeline.txt 2>&1; tail -1 gpurun_out/r4n_timeline.txt
timeout 900 python bench.py --steps 30 --warmup 5 --no-secondary --no-cpu-baseline > gpurun_out/r4n_bench.json 2> gpurun_out/r4n_bench.err; echo bench rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/r4n_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d.get('graphed',{}).get('ms_per_step'), d['e2e']['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r4n_launches.csv python scripts/diag_step.py > gpurun_out/r4n_ncu_launch.log 2>&1; echo launch rc=$?
