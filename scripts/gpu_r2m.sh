mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_expansion.py tests/test_gpu_geometry.py tests/test_gpu_rays.py -q -x 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2m_launches.csv python scripts/diag_step.py > gpurun_out/r2m_ncu_launch.log 2>&1; echo launch rc=$?
python scripts/ncu_launch_summary.py gpurun_out/r2m_launches.csv | head -12
