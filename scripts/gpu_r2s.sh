mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_expansion.py tests/test_gpu_multiprocess.py tests/test_gpu_rho6.py tests/test_gpu_geometry.py -q -x 2>&1 | tail -2
timeout 500 python scripts/diag_dev_timeline.py 2>&1 | grep -v "^\s*$" | grep -v Warn | sed -n 3,80p | awk '{print $1, $2, $3, $6}' | cut -c1-90
timeout 600 python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/r2s_bench.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2s_bench.json'));print('bench', d['ms_per_step'], d['graphed']['ms_per_step'])"
