set -x
timeout 300 python -m pytest tests/test_gpu_expansion.py -q -k "m2m_l2l_m2l or tensor_core or cfg1 or config2 or golden or torch_io" 2>&1 | tail -15
