cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prof_i8.py > gpurun_out/prof_i8_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused8_i8 -s 2 -c 1 -o gpurun_out/prof_i8 python scripts/prof_i8.py > gpurun_out/ncu_i8.log 2>&1
