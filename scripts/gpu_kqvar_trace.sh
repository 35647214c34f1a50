# time k_fused8_q variants (VARS="name ...", build/<name>/libdctf_var.so from build_var.sh) on config 5 and print the
# clock64 pipeline trace of QDBG builds (QV="name ..."); output in gpurun_out/kqvar_trace.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(KQ_TIMEOUT=60 VARS="${VARS}" bash scripts/gpu_kqvar.sh
for q in ${QV}; do echo "== trace $q"; DCTF_LIB_PATH=build/$q/libdctf_var.so timeout 120 python scripts/kq_trace3.py 2>&1 | tail -9; done) > gpurun_out/kqvar_trace.log 2>&1
cat gpurun_out/kqvar_trace.log
