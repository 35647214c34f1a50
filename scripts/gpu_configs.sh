cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-cfg}
timeout 2400 python -m pytest tests/test_gpu_configs.py -m gpu -q -s --timeout 1800 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
