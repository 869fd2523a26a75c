timeout 300 python scripts/diag_l2p.py > gpurun_out/plain_l2p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:l2p_kernel -s 8 -c 2 \
  -o gpurun_out/prof_l2p python scripts/diag_l2p.py > gpurun_out/ncu_l2p.log 2>&1; echo ncu rc=$?
