mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_expansion.py -q -x -k "separable_far" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_expansion.py tests/test_gpu_geometry.py -q -x 2>&1 | tail -5
timeout 900 python bench.py --steps 30 --warmup 5 --no-secondary --no-cpu-baseline > gpurun_out/r4d_bench.json 2> gpurun_out/r4d_bench.err; echo bench rc=$?
tail -2 gpurun_out/r4d_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r4d_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d.get('graphed',{}).get('ms_per_step'), d['e2e']['ms_per_step'])"
timeout 300 python scripts/diag_dev_timeline.py > gpurun_out/r4d_timeline.txt 2>&1
