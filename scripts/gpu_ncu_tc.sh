cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prof_tc.py > gpurun_out/prof_tc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 2 -c 1 -o gpurun_out/prof_tc16 python scripts/prof_tc.py > gpurun_out/ncu_tc16.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 6 -c 1 -o gpurun_out/prof_tc8 python scripts/prof_tc.py > gpurun_out/ncu_tc8.log 2>&1
