mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo bench rc=$?; tail -2 gpurun_out/r2g_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2g_bench_ref.json 2> gpurun_out/r2g_bench_ref.err; echo ref rc=$?
timeout 900 python bench.py --config 5 --steps 4 --warmup 3 > gpurun_out/r2g_bench_cfg5.json 2> gpurun_out/r2g_bench_cfg5.err; echo cfg5 rc=$?
