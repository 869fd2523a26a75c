mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rays.py tests/test_gpu_training_loops.py tests/test_gpu_autograd.py -q -x 2>&1 | tail -2
timeout 600 python scripts/diag_cfg4.py 2>&1 | tail -4 | cut -c1-600
