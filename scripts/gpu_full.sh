set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?; tail -3 gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?; tail -3 gpurun_out/bench_ref.err
nproc; lscpu | grep "Model name"
