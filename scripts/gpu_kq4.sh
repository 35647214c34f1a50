timeout 900 python -m pytest tests/test_gpu_kq.py -x -q 2>&1 | tail -2
DCTF_LIB_PATH=paper_1710_07193_b200/libdctf_b200.so timeout 120 python scripts/kq_var.py 2>&1 | tail -2
