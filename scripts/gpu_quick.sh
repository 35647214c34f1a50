# usage: bash scripts/gpu_quick.sh <tag> [bench args]  -> gpu tests + short bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-q}; shift
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
