timeout 600 python -m pytest tests/test_gpu_rays.py -q 2>&1 | tail -30
