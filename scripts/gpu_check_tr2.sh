# 2-rank code path of bench.py on the one-GPU box (gloo; ranks share the GPU: a code-path check, not a timing)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
DCTF_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tr2.json 2> gpurun_out/bench_tr2.err; echo "tr2 rc=$?"
timeout 600 python bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_ref_tr2.json 2> gpurun_out/bench_ref_tr2.err; echo "ref tr2 rc=$?"
tail -2 gpurun_out/bench_tr2.err; head -c 400 gpurun_out/bench_tr2.json; echo; head -c 300 gpurun_out/bench_ref_tr2.json
