# Accountant fencing once per batch of mailbox entries; entry-major reshard; strided-slice micro-benchmark.
set -x
python -m pytest tests/test_gpu_heads.py tests/test_gpu_concurrency.py tests/test_gpu_batch.py -q -x -p no:cacheprovider 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "litmus or signal" 2>&1 | tail -2
W="--work c2batch,t4prime,l2req --cand plain=0:0:0:0:0 --cand sig=0:0:0:0:0:1"
AB_TAG=accbatch python scripts/engine_ab.py $W 2>&1 | tail -6
python scripts/reshard_sweep.py --quick --out gpurun_out/reshard_r02e.json 2>&1 | cut -c1-200 | tail -12
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/copy_micro scripts/native/copy_micro.cu && timeout 300 /tmp/copy_micro F > gpurun_out/copy_micro_rows.jsonl; cat gpurun_out/copy_micro_rows.jsonl
