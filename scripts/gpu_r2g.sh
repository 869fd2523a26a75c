mkdir -p gpurun_out
timeout 900 python scripts/diag_bench_seq.py > gpurun_out/seq.log 2>&1
grep -n "fc2t2:\|Error\|File" gpurun_out/seq.log | head -30
