for v in build/exp1/libdctf_var.so build/exp3/libdctf_var.so paper_1710_07193_b200/libdctf_b200.so; do
  DCTF_LIB_PATH=$v timeout 120 python scripts/kq_var.py 2>&1 | tail -2
done
