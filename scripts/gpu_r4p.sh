mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_expansion.py tests/test_gpu_geometry.py -q -x 2>&1 | tail -2
ALT=paper_2111_00110_b200/build_ab/lib_epi.so bash scripts/gpu_ab3.sh
