mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_expansion.py tests/test_gpu_geometry.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r3c_bench.json 2> gpurun_out/r3c_bench.err; echo bench rc=$?
tail -2 gpurun_out/r3c_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r3c_launches.csv python scripts/diag_step.py > gpurun_out/r3c_ncu_launch.log 2>&1; echo launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"brick_scatter_rank|brick_p2m|brick_hist" -o /tmp/r3c_brick python scripts/diag_step.py > gpurun_out/r3c_ncu_brick.log 2>&1; echo brick rc=$?
ncu -i /tmp/r3c_brick.ncu-rep --page details --csv > gpurun_out/r3c_brick_details.csv 2>/dev/null
for k in brick_scatter_rank brick_p2m brick_hist; do
  ncu -i /tmp/r3c_brick.ncu-rep --page source --csv --print-source sass --kernel-name regex:$k --launch-skip 1 --launch-count 1 > gpurun_out/r3c_sass_$k.csv 2> gpurun_out/r3c_sass_$k.err; echo sass $k rc=$?
done
ls -la gpurun_out/ | grep r3c
