# headline evidence for k_fused8_sep: bench line, headline launch list, ncu capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r04g.json 2> gpurun_out/bench_r04g.err; echo "bench rc=$?" >> gpurun_out/bench_r04g.err
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_headline_r04g.csv $CMD > /dev/null 2>&1
KERNELS="k_fused8_sep" bash scripts/gpu_ncu_all.sh r04g
