# full GPU suite (unit + configs) then bench; usage: bash scripts/gpu_all.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-all}
timeout 3000 python -m pytest tests -m gpu -q -s --timeout 2400 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
