mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vol_seg_payload|vol_segments|vol_forward" -c 3 -o gpurun_out/r2y_vol python scripts/diag_cfg4.py > gpurun_out/r2y_ncu.log 2>&1; echo full rc=$?
