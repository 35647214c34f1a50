# k_fused8_q on the config-5 bench: plain run, launch list, one ncu --set full capture
# usage: bash scripts/gpu_prof_q.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-q}
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err || { tail gpurun_out/plain_$TAG.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_fused8_q$" -s 1 -c 1 \
    -o gpurun_out/prof_k_fused8_q_$TAG $CMD > gpurun_out/ncu_k_fused8_q_$TAG.log 2>&1
echo "ncu rc=$?"
