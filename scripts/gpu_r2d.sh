set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -25
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -25
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo bench rc=$?
tail -3 gpurun_out/r2d_bench.err
timeout 600 python bench.py --config 5 --steps 4 --warmup 3 > gpurun_out/r2d_cfg5.json 2> gpurun_out/r2d_cfg5.err; echo cfg5 rc=$?
tail -3 gpurun_out/r2d_cfg5.err
