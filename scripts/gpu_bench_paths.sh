# bench entry paths: torchrun N=1, reference arm (also under torchrun)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo "rc=$?" >> gpurun_out/bench_torchrun.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench_ref_tr.json 2> gpurun_out/bench_ref_tr.err; echo "rc=$?" >> gpurun_out/bench_ref_tr.err
# multi-rank code path (2 ranks sharing the one GPU, gloo; timings not valid)
DCTF_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline --no-aux > gpurun_out/bench_tr2.json 2> gpurun_out/bench_tr2.err; echo "rc=$?" >> gpurun_out/bench_tr2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_ref_tr2.json 2> gpurun_out/bench_ref_tr2.err; echo "rc=$?" >> gpurun_out/bench_ref_tr2.err
