# time k_fused8_q measurement variants on config 5 (scripts/build_var.sh builds them)
for v in ${VARS:-default v1 v3 v5 v6}; do
  if [ $v = default ]; then L=paper_1710_07193_b200/libdctf_b200.so; else L=build/$v/libdctf_var.so; fi
  echo -n "$v: "; DCTF_LIB_PATH=$L timeout ${KQ_TIMEOUT:-90} python scripts/kq5_time.py 2>&1 | tail -1
done
