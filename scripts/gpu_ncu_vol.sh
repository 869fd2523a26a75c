POSES=2 timeout 300 python scripts/diag_cfg4.py > gpurun_out/plain_cfg4.log 2>&1 && \
POSES=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"vol_payload|vol_forward|vol_totals|insert_sorted|depth_walk" -s 4 -c 4 \
  -o gpurun_out/prof_vol python scripts/diag_cfg4.py > gpurun_out/ncu_vol.log 2>&1; echo ncu rc=$?
grep CFG4 gpurun_out/plain_cfg4.log
