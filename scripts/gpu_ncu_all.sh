# ncu evidence for every kernel on its bench workload (one ncu tool per call).
# usage: bash scripts/gpu_ncu_all.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
for K in ${KERNELS:-k_fused8_sep k_fused8_sym k_fused8 k_fused8_i8 k_coef8_sep k_fused16_sep k_fused16_sym k_fused16 k_coef8_sym k_coef8 k_coef16_sep k_coef16_sym k_coef16 k_coef_split3}; do
  ncu --set full --clock-control none --import-source on -k regex:"^${K}$" -s 1 -c 1 \
      -o gpurun_out/prof_${K}_$TAG $CMD > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
echo done
