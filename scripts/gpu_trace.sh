for v in ${VARS:-qdbg}; do echo "== $v"; DCTF_LIB_PATH=build/$v/libdctf_var.so timeout 300 python scripts/kq_trace.py 2>&1 | grep -A1 "CTA 0\|mean stage" | head -5; done
