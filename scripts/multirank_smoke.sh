# Functional check of the N > 1 code paths on a ONE-GPU box: N ranks share cuda:0 through
# CUDA IPC (gloo process group), reduced pools.  Not a measurement — every "peer" is the same GPU.
# Off by default: ranks that are separate processes on one GPU are not guaranteed to be
# co-scheduled (B200_PROFILING: Xid 109 under context switching), so a rank whose kernel waits
# on another rank's flag could hang the box.  The N > 1 host logic is covered on the CPU
# (tests/test_dist_gloo.py, gloo world 2); set DYNA_MULTIRANK_ONE_GPU=1 to run it anyway.
if [ "${DYNA_MULTIRANK_ONE_GPU:-0}" != "1" ]; then echo "multirank_smoke: skipped (one-GPU box)"; exit 0; fi
export DYNA_BENCH_SAME_DEVICE=1 DYNA_BENCH_BACKEND=gloo DYNA_BENCH_SMALL=1
for n in 2 3; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29517 + n)) bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29530 scripts/allpairs.py --num-blocks 2000 --steps 3 --warmup 1 --check 2>&1 | tail -2
