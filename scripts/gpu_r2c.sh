set -x
python -m paper_2111_00110_b200.build
timeout 600 python -m pytest tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -25
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo bench rc=$?
tail -3 gpurun_out/r2c_bench.err
timeout 600 python bench.py --config 5 --steps 4 --warmup 2 > gpurun_out/r2c_cfg5.json 2> gpurun_out/r2c_cfg5.err; echo cfg5 rc=$?
tail -3 gpurun_out/r2c_cfg5.err
