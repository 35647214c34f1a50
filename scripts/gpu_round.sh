# round evidence: full GPU suite, default bench line, reference arm, headline launch list,
# ncu --set full of the headline kernel (k_fused8_q, bench config 5). usage: bash scripts/gpu_round.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r07}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_fused8_q$" -s 3 -c 1 \
    -o gpurun_out/prof_k_fused8_q_$TAG $CMD > gpurun_out/ncu_q_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log; head -c 600 gpurun_out/bench_$TAG.json
