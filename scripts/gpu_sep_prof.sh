REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sep_pass -c 3 \
  -o gpurun_out/sep_prof python scripts/diag_sep.py > gpurun_out/ncu_sep.log 2>&1; echo ncu rc=$?
