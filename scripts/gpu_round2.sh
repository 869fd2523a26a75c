# round-2 evidence at HEAD: GPU tests, smoke, one-step ncu captures (launch
# list, --set full -> traffic.json), bench (+ reference arm)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2f_pytest_gpu.log 2>&1; tail -2 gpurun_out/r2f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python scripts/diag_step.py > gpurun_out/r2f_diag_step.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2f_launches.csv python scripts/diag_step.py > gpurun_out/r2f_ncu_launch.log 2>&1; echo launch rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -o /tmp/r2f_step_full python scripts/diag_step.py > gpurun_out/r2f_ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_traffic.py /tmp/r2f_step_full.ncu-rep 1 gpurun_out/r2f_traffic.json > /dev/null; echo traffic rc=$?
cp gpurun_out/r2f_traffic.json profiles/traffic.json
ncu -i /tmp/r2f_step_full.ncu-rep --page details --csv > gpurun_out/r2f_step_details.csv 2>/dev/null; echo details rc=$?
ncu -i /tmp/r2f_step_full.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum > gpurun_out/r2f_step_raw.csv 2>/dev/null; echo raw rc=$?
timeout 300 python scripts/diag_timeline.py > gpurun_out/r2f_timeline.txt 2>&1; tail -1 gpurun_out/r2f_timeline.txt
timeout 1500 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo bench rc=$?; tail -2 gpurun_out/r2f_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err; echo ref rc=$?
du -sh gpurun_out
