mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo bench rc=$?
tail -2 gpurun_out/r2z_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2z_launches.csv python scripts/diag_step.py > gpurun_out/r2z_ncu_launch.log 2>&1; echo launch rc=$?
timeout 1200 ncu --set full --clock-control none --profile-from-start off -o /tmp/r2z_step_full python scripts/diag_step.py > gpurun_out/r2z_ncu_full.log 2>&1; echo full rc=$?
python scripts/ncu_traffic.py /tmp/r2z_step_full.ncu-rep 1 gpurun_out/r2z_traffic.json > /dev/null; echo traffic rc=$?
ncu -i /tmp/r2z_step_full.ncu-rep --page details --csv > gpurun_out/r2z_step_details.csv 2>/dev/null; echo details rc=$?
timeout 600 python -m pytest tests/test_gpu_rays.py -q -s -k config3 2>&1 | grep -i "config\|adjoint\|backward\|passed\|failed" | head
timeout 900 python bench.py --config 5 --steps 4 --warmup 3 > gpurun_out/r2z_cfg5.json 2> gpurun_out/r2z_cfg5.err; echo cfg5 rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2z_ref.json 2> gpurun_out/r2z_ref.err; echo ref rc=$?
python scripts/ncu_traffic.py /tmp/r2z_step_full.ncu-rep 1 gpurun_out/r2z_traffic.json > /dev/null; echo traffic2 rc=$?
