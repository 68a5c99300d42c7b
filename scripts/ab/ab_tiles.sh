# A/B of the tile engine's knobs on the quick reshard cases (one_launch + calls, tiles only).
set -x
DYNA_KV_TILE_RR=1 timeout 600 python -m pytest tests/test_gpu_heads.py -q -x -p no:cacheprovider -k "reshard" 2>&1 | tail -1
for v in "base:" "rr:DYNA_KV_TILE_RR=1" "b16k:DYNA_KV_TILE_BYTES=16384" "b64k:DYNA_KV_TILE_BYTES=65536" \
         "l2none:DYNA_KV_TILE_L2=0" "l2_128:DYNA_KV_TILE_L2=2" "rr_b16k:DYNA_KV_TILE_RR=1 DYNA_KV_TILE_BYTES=16384" "base2:"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/reshard_sweep.py --quick --engines tiles --out gpurun_out/ab_tiles_$name.json > /dev/null 2>&1
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
r = json.load(open(f"gpurun_out/ab_tiles_{n}.json"))["results"]
print(n, " ".join(f"{x['model'][:5]}{x['tp_src']}>{x['tp_dst']}{x['mode'][0]}={x['frac_of_measured_hbm']:.3f}" for x in r))
PY
done
