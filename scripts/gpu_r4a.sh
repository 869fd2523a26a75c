mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4a_pytest_gpu.log 2>&1; tail -3 gpurun_out/r4a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err; echo bench rc=$?; tail -2 gpurun_out/r4a_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r4a_launches.csv python scripts/diag_step.py > gpurun_out/r4a_ncu_launch.log 2>&1; echo launch rc=$?
