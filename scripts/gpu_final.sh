# end-of-round evidence: full GPU suite, default bench line, headline launch list, ncu of every kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-final}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_headline_$TAG.csv $CMD > /dev/null 2>&1
bash scripts/gpu_ncu_all.sh $TAG
