# Round 2: dyna_kv_reshard (one interleaved launch) vs per-pair calls; signalled vs unsignalled
# ring; ncu captures of the ring (c2, t4) and rows kernels.
set -x
python -m pytest tests/test_gpu_heads.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider 2>&1 | tail -4
python scripts/reshard_sweep.py --out gpurun_out/reshard_r02b.json 2>&1 | cut -c1-200 | tail -30
AB_TAG=sig python scripts/engine_ab.py --work c2batch,t4prime,l2req --cand plain=0:0:0:0:0 --cand sig=0:0:0:0:0:1 2>&1 | tail -8
bash scripts/gpu_r02_ncu.sh 2>&1 | tail -12
