for r in 1 2; do
for v in 0 1; do
  FC2T2_SERIAL_CASCADE=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('serial=$v', round(d['ms_per_step'],4), 'graphed', round(d['graphed']['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],3))"
done; done
