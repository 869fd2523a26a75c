mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"brick_scatter_rank" -o gpurun_out/r2r_brick python scripts/diag_step.py > gpurun_out/r2r_ncu.log 2>&1; echo full rc=$?
ls -la gpurun_out
