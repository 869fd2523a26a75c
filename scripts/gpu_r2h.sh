mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo bench rc=$?
tail -3 gpurun_out/r2h_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2h_launches.csv python scripts/diag_step.py > gpurun_out/r2h_ncu_launch.log 2>&1; echo launch rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -o /tmp/r2h_step_full python scripts/diag_step.py > gpurun_out/r2h_ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_traffic.py /tmp/r2h_step_full.ncu-rep 1 gpurun_out/r2h_traffic.json > /dev/null; echo traffic rc=$?
ncu -i /tmp/r2h_step_full.ncu-rep --page details --csv > gpurun_out/r2h_step_details.csv 2>/dev/null; echo details rc=$?
ls -la gpurun_out
