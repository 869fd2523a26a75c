set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench rc=$?
tail -2 gpurun_out/bench3.err
