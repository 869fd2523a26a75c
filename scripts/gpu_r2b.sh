set -x
python -m paper_2111_00110_b200.build
timeout 900 python -m pytest tests/test_gpu_expansion.py -q -x -k "brick or stable_counting or explicit or recycling" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_geometry.py -q -s 2>&1 | tail -8
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench rc=$?
tail -3 gpurun_out/r2b_bench.err
