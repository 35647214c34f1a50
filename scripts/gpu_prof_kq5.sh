# one ncu --set full capture of k_fused8_q on config 5 (scripts/kq5_time.py workload)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-x}
ncu --set full --clock-control none --import-source on -k regex:"^k_fused8_q$" -s 3 -c 1 \
    -o gpurun_out/prof_kq5_$TAG python scripts/kq5_time.py > gpurun_out/ncu_kq5_$TAG.log 2>&1
echo "ncu rc=$?"
