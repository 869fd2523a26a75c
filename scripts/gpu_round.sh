# round evidence: GPU tests, bench (+reference arm), one-step ncu captures -> traffic.json
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python scripts/diag_step.py > gpurun_out/diag_step.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --profile-from-start off -o gpurun_out/step_traffic \
  python scripts/diag_step.py > gpurun_out/ncu_step.log 2>&1; echo ncu rc=$?
python scripts/ncu_traffic.py gpurun_out/step_traffic.ncu-rep 1 gpurun_out/traffic.json > /dev/null 2>&1; echo traffic rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:${TOPK:-l2p_warp} -c 2 -o gpurun_out/top_full python scripts/diag_step.py > gpurun_out/ncu_top.log 2>&1; echo ncu top rc=$?
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?; tail -2 gpurun_out/bench_full.err
if [ -n "$REF" ]; then timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?; fi
du -sh gpurun_out
