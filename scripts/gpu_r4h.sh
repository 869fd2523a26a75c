mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"sep_pass_kernel|sep_pre|sep_post" -c 12 -o /tmp/r4h_sep python scripts/diag_step.py > gpurun_out/r4h_ncu.log 2>&1; echo sep rc=$?
ncu -i /tmp/r4h_sep.ncu-rep --page details --csv > gpurun_out/r4h_sep_details.csv 2>/dev/null
for id in 1 2 3; do
  ncu -i /tmp/r4h_sep.ncu-rep --page source --csv --print-source sass --launch-skip $id --launch-count 1 > gpurun_out/r4h_sass_$id.csv 2> gpurun_out/r4h_sass_$id.err; echo sass $id rc=$?
done
