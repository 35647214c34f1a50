cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(for i in 0 1 2 3; do echo "== all frames on plan $i"; KQ_IDX=$i timeout 90 python scripts/kq5_time.py 2>&1 | tail -1; done
for i in 0 1; do echo "== trace plan $i"; KQ_IDX=$i DCTF_LIB_PATH=build/rq/libdctf_var.so timeout 120 python scripts/kq_trace3.py 2>&1 | tail -9; done) > gpurun_out/s10.log 2>&1
cat gpurun_out/s10.log
