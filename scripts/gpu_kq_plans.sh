# time k_fused8_q variants (VARS, build/<name>/libdctf_var.so) on config 5 and on single-plan 64-frame batches (IDXS="" 0 1 2 3:
# KQ_IDX of scripts/kq5_time.py), and trace QDBG builds (QV) per plan; output in gpurun_out/s11.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(for v in $VARS; do for i in ${IDXS:-"" 0 1}; do echo -n "$v plan[$i] "; KQ_IDX=$i DCTF_LIB_PATH=build/$v/libdctf_var.so timeout 90 python scripts/kq5_time.py 2>&1 | tail -1 | cut -c1-150; done; done
for q in $QV; do for i in 0 1; do echo "== trace $q plan $i"; KQ_IDX=$i DCTF_LIB_PATH=build/$q/libdctf_var.so timeout 120 python scripts/kq_trace3.py 2>&1 | tail -9; done; done) > gpurun_out/s11.log 2>&1
cat gpurun_out/s11.log
