# Multi-GPU evidence (needs >= 2 GPUs on one node; nothing here runs on a one-GPU box).
# NVLink forms of the path: bench.py at N = 2 (the 4' pair target) and N = 4/8 (configs[4] all
# pairs vs the load-aware bound), each line with the NCCL send/recv baseline (B1) on the same
# bytes; the cross-GPU parity tests; peer calibration entries; the overlap experiment with the
# destination on another GPU.
set -x
N=$(nvidia-smi -L | wc -l)
if [ "$N" -lt 2 ]; then echo "gpu_multi.sh: $N GPU visible, nothing to do"; exit 0; fi
for n in 2 4 8; do
  [ $n -le $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n --no-cpu-baseline > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  cat gpurun_out/bench_n$n.json
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) scripts/allpairs.py --steps 5 --warmup 2 --check 2>&1 | tail -2
done
python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 2700 python scripts/calibrate.py --peer --out gpurun_out/calibration_peer.json --inc gpurun_out/calib_peer.inc \
    > gpurun_out/calibrate_peer.log 2>&1; tail -1 gpurun_out/calibrate_peer.log
timeout 1800 python scripts/overlap.py --dst-device 1 --chunks 1024,4096 --budgets 0,16 --layers \
    --out gpurun_out/overlap_nvlink.json 2>&1 | tail -4
