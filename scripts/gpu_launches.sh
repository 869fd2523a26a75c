# launch list (cold-cache, serialised under ncu) of one headline bench run
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/plain_launch.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
