mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; echo bench rc=$?
tail -2 gpurun_out/r3a_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r3a_launches.csv python scripts/diag_step.py > gpurun_out/r3a_ncu_launch.log 2>&1; echo launch rc=$?
timeout 1200 ncu --set full --clock-control none --profile-from-start off -o /tmp/r3a_step_full python scripts/diag_step.py > gpurun_out/r3a_ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_traffic.py /tmp/r3a_step_full.ncu-rep 1 gpurun_out/r3a_traffic.json > /dev/null; echo traffic rc=$?
ncu -i /tmp/r3a_step_full.ncu-rep --page details --csv > gpurun_out/r3a_step_details.csv 2>/dev/null; echo details rc=$?
