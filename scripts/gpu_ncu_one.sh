# usage: bash scripts/gpu_ncu_one.sh <kernel> <tag>  -> one ncu --set full capture on the bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
K=$1; TAG=${2:-x}
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"^${K}$" -s 1 -c 1 \
    -o gpurun_out/prof_${K}_$TAG $CMD > gpurun_out/ncu_${K}_$TAG.log 2>&1
