mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:l2p_kernel -c 2 -o gpurun_out/r2o_l2p python scripts/diag_l2p_ab.py > gpurun_out/r2o_ncu.log 2>&1; echo rc=$?
