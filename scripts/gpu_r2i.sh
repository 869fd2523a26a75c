mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo bench rc=$?
tail -3 gpurun_out/r2i_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2i_launches.csv python scripts/diag_step.py > gpurun_out/r2i_ncu_launch.log 2>&1; echo launch rc=$?
