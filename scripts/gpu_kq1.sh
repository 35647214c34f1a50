set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 120 python scripts/kq_smoke.py 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_kq.py -x -q 2>&1 | tail -15
timeout 300 python scripts/kq_time.py 2>&1 | tail -12
