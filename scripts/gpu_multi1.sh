timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_cpp.py tests/test_gpu_kq.py -x -q 2>&1 | tail -15
