# round-4 evidence: PDL tests, headline launch list (--no-aux), ncu captures of every kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pdl.py -q > gpurun_out/pytest_pdl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pdl.log
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_headline_r04.csv $CMD > /dev/null 2>&1
bash scripts/gpu_ncu_all.sh r04
