timeout 300 python scripts/diag_sort.py 2>&1 | grep SORT_MS && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"radix_scatter|radix_hist|cell_keys" -s 6 -c 3 \
  -o gpurun_out/prof_sort python scripts/diag_sort.py > gpurun_out/ncu_sort.log 2>&1; echo ncu rc=$?
