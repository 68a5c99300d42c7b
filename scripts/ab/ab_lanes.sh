# VEC warp-cooperative decode (k_copy_lanes, 2 CTAs/SM) vs round-1 k_copy_vec (3 CTAs/SM); lane-parallel
# decode in k_copy_rows vs round 1 (profiles/r01_reshard_final.json).  Parity first.
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_heads.py tests/test_gpu_fuzz.py tests/test_gpu_batch.py -q -x -p no:cacheprovider 2>&1 | tail -4
C="--cand vec8=1:8192:0:8:0 --cand vec16k=1:16384:0:8:0 --cand vec4k=1:4096:0:8:0 --cand vec_u16=1:16384:0:16:0"
DYNA_KV_LANES=0 AB_TAG=lanes0 python scripts/engine_ab.py $C 2>&1 | tail -20
AB_TAG=lanes1 python scripts/engine_ab.py $C 2>&1 | tail -20
python scripts/reshard_sweep.py --out gpurun_out/reshard_r02.json 2>&1 | tail -20
