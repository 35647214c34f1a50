# usage: bash scripts/gpu_ncu.sh <tag>   (one ncu tool per gpurun call)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused8 -s 3 -c 1 -o gpurun_out/prof_fused8_$TAG $CMD > gpurun_out/ncu_full_fused8_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_coef8 -s 3 -c 1 -o gpurun_out/prof_coef8_$TAG $CMD > gpurun_out/ncu_full_coef8_$TAG.log 2>&1
echo done
