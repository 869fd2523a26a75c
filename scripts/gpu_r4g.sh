mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"brick_scatter_rank|brick_p2m|brick_hist" -o /tmp/r4g_brick python scripts/diag_step.py > gpurun_out/r4g_ncu_brick.log 2>&1; echo brick rc=$?
ncu -i /tmp/r4g_brick.ncu-rep --page details --csv > gpurun_out/r4g_brick_details.csv 2>/dev/null
for k in brick_scatter_rank brick_p2m; do
  ncu -i /tmp/r4g_brick.ncu-rep --page source --csv --print-source sass --kernel-name regex:$k --launch-skip 1 --launch-count 1 > gpurun_out/r4g_sass_$k.csv 2> gpurun_out/r4g_sass_$k.err; echo sass $k rc=$?
done
ls -la gpurun_out/ | grep r4g
