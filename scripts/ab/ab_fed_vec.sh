# VEC engine through the decoder-fed row kernel (DYNA_KV_FED_VEC=1) vs k_copy_lanes.
set -x
DYNA_KV_FED_VEC=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider 2>&1 | tail -2
C="--work l2req,c2batch,t4prime,c3c512,q8 --cand auto=0:0:0:0:0 --cand vec8=1:8192:0:8:0 --cand vec4k=1:4096:0:8:0 --cand vec16k=1:16384:0:8:0"
AB_TAG=fed0 python scripts/engine_ab.py $C 2>&1 | tail -3
DYNA_KV_FED_VEC=1 AB_TAG=fed1 python scripts/engine_ab.py $C 2>&1 | tail -3
