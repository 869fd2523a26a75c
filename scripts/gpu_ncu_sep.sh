# separable M2L: event timings, then one ncu --set full capture of each sep kernel
timeout 300 python scripts/diag_sep.py 2>&1 | tail -6
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sep_ -c 5 \
  -o gpurun_out/sep_full python scripts/diag_sep.py > gpurun_out/ncu_sep.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_sep.log
