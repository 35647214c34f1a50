# headline bench (N=1), the reference arm, and the 2-rank code path (gloo, ranks sharing the GPU)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
DCTF_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-aux --no-cpu-baseline > gpurun_out/bench_tr2.json 2> gpurun_out/bench_tr2.err; echo "tr2 rc=$?"
tail -3 gpurun_out/bench.err
