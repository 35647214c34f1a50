cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for l in paper_1710_07193_b200/libdctf_b200.so scratch_libs/lib_xs4.so scratch_libs/lib_xs6.so; do echo "$l"; DCTF_LIB_PATH=$PWD/$l timeout 300 python scripts/tc_time.py; done > gpurun_out/tc_sweep.log 2>&1
