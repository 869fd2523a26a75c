mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"sep_pass_kernel" -c 3 -o gpurun_out/r2w_sep python scripts/diag_step.py > gpurun_out/r2w_ncu.log 2>&1; echo full rc=$?
