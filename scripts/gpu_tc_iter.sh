timeout 600 python scripts/diag_tc.py 2>&1 | grep -E "^L|Error"
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench rc=$?; tail -2 gpurun_out/bench4.err
