timeout 600 python -m pytest tests/test_gpu_rays.py -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench rc=$?; tail -3 gpurun_out/bench7.err
