set -x
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/diag_p2m_l4.py 2>&1 | tail -12
timeout 300 python scripts/ubench/peaks.py r2 2>&1 | tail -3
cp profiles/r2_peaks.json gpurun_out/ 
