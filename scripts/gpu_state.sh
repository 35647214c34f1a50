# round-2 state check: full GPU suite, default bench line, reference arm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-state}
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.err
tail -2 gpurun_out/pytest_$TAG.log; cat gpurun_out/bench_$TAG.json | head -c 3000
