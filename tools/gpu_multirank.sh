# Multi-rank bench path on one GPU (gloo process group, both ranks on GPU 0):
# checks sharding offsets, barrier / max-over-ranks timing and the JSON line.
cd $GRAFT_REPO_ROOT
DK_BENCH_SAME_DEVICE=1 DK_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 40 --warmup 5 --no-cpu --e2e-steps 100 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo "rc=$?" >> gpurun_out/bench_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_ref_2rank.json 2> gpurun_out/bench_ref_2rank.err
echo "rc=$?" >> gpurun_out/bench_ref_2rank.err
