# Decoder-fed head-sliced kernel: parity (heads, channel heads, fuzz), then the reshard sweep.
set -x
python -m pytest tests/test_gpu_heads.py tests/test_gpu_channel.py tests/test_gpu_fuzz.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider 2>&1 | tail -3
python scripts/reshard_sweep.py --out gpurun_out/reshard_r02f.json 2>&1 | cut -c1-200 | tail -30
