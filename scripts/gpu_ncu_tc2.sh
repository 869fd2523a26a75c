# ncu --set full of the config-2 level-5 tcgen05 M2L launch (8th m2l_tc launch of diag_tc_time.py)
timeout 300 python scripts/diag_tc_time.py > gpurun_out/plain_tc2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:m2l_tc_kernel -s ${SKIP:-7} -c 1 \
  -o gpurun_out/prof_m2l_tc2 python scripts/diag_tc_time.py > gpurun_out/ncu_tc2.log 2>&1; echo ncu rc=$?
