mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --profile-from-start off -o /tmp/r2v_step_full python scripts/diag_step.py > gpurun_out/r2v_ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_traffic.py /tmp/r2v_step_full.ncu-rep 1 gpurun_out/r2v_traffic.json > /dev/null; echo traffic rc=$?
ncu -i /tmp/r2v_step_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum > gpurun_out/r2v_raw.csv 2>/dev/null; echo raw rc=$?
