set -x
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench rc=$?
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_p.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncu_launch rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"depth_walk|vol_payload|vol_forward|radix_scatter|l2p_kernel|p2m_sorted" -c 8 -o gpurun_out/prof_r1c_misc python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_misc.log 2>&1; echo ncu_full rc=$?
