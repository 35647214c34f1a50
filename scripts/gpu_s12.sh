cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export KQ_IDX=${KQ_IDX:-0}
ncu --set full --clock-control none --import-source on -k regex:"^k_fused8_q$" -s 3 -c 1 \
    -o gpurun_out/prof_kq5_light python scripts/kq5_time.py > gpurun_out/ncu_kq5_light.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_kq5_light.ncu-rep --page source --csv > gpurun_out/prof_kq5_light_source.csv 2>/dev/null
