mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"brick_scatter|brick_p2m" -o gpurun_out/r2n_brick python scripts/diag_step.py > gpurun_out/r2n_ncu.log 2>&1; echo full rc=$?
ls -la gpurun_out
timeout 600 python -m pytest tests/test_gpu_expansion.py tests/test_gpu_geometry.py tests/test_gpu_rays.py -q -x 2>&1 | tail -3
