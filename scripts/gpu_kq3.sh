timeout 900 python -m pytest tests/test_gpu_kq.py -x -q 2>&1 | tail -3
timeout 300 python scripts/kq_time.py 2>&1 | tail -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused8_q --launch-skip 2 -c 1 -o gpurun_out/kq_cfg2b python scripts/kq_prof.py > gpurun_out/kq_ncu.log 2>&1; tail -1 gpurun_out/kq_ncu.log
