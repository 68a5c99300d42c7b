# Functional check of the N > 1 code paths on a ONE-GPU box: two ranks share cuda:0 through
# CUDA IPC (gloo process group).  Not a measurement — both "peers" are the same GPU.
export DYNA_BENCH_SAME_DEVICE=1 DYNA_BENCH_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --steps 50 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29518 scripts/allpairs.py --num-blocks 2000 --steps 3 --warmup 1 --check 2>&1 | tail -2
