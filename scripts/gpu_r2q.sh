timeout 300 python scripts/diag_cfg1.py 2>&1 | tail -1 | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_expansion.py tests/test_gpu_training_loops.py tests/test_gpu_rays.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2q_launches.csv python scripts/diag_step.py > /dev/null 2>&1; echo launch rc=$?
python scripts/ncu_launch_summary.py gpurun_out/r2q_launches.csv 2>/dev/null | head -6
