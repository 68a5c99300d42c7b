# Ring (decoder-fed BULK) vs round-1 engines on the headline workloads.
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -5
C="--cand auto=0:0:0:0:0 --cand bulk6=2:32768:6:0:0 --cand bulk4=2:32768:4:0:0 --cand vec2=1:8192:0:8:296 --cand vec3=1:8192:0:8:0 --cand vec2p16=1:16384:0:8:296"
DYNA_KV_RING=0 AB_TAG=ring0 python scripts/engine_ab.py $C 2>&1 | tail -40
AB_TAG=ring_lagdef python scripts/engine_ab.py $C --cand bulk8=2:24576:8:0:0 2>&1 | tail -40
DYNA_KV_LAG=1 AB_TAG=ring_lag1 python scripts/engine_ab.py --cand bulk6=2:32768:6:0:0 --cand bulk4=2:32768:4:0:0 --cand bulk3=2:32768:3:0:0 2>&1 | tail -20
