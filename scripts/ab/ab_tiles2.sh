# Tile engine, device-bound sizes (s = 16384: ~2 GiB per Llama-3-8B reshard, host cost << device time):
# entry-major vs round-robin, 128-B vs 256-B L2 promotion; rows engine beside.
set -x
DYNA_KV_TILE_RR=1 timeout 600 python -m pytest tests/test_gpu_heads.py -q -x -p no:cacheprovider -k "reshard" 2>&1 | tail -1
for v in "base:" "rr:DYNA_KV_TILE_RR=1" "base2:" "rr2:DYNA_KV_TILE_RR=1"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/reshard_sweep.py --quick --s 16384 --chunk 1024 --engines tiles --reps 10 --out gpurun_out/ab2_tiles_$name.json > /dev/null 2>&1
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
r = json.load(open(f"gpurun_out/ab2_tiles_{n}.json"))["results"]
print(n, " ".join(f"{x['model'][:5]}{x['tp_src']}>{x['tp_dst']}{x['mode'][0]}={x['frac_of_measured_hbm']:.3f}/h{x['host_ms_per_reshard']:.2f}/d{x['ms']:.2f}" for x in r))
PY
done
# timeout 600 python scripts/reshard_sweep.py --quick --s 16384 --chunk 1024 --engines rows --reps 10 --out gpurun_out/ab2_rows.json > /dev/null 2>&1
python - <<'PY'
import json
r = json.load(open("gpurun_out/ab2_rows.json"))["results"]
print("rows", " ".join(f"{x['model'][:5]}{x['tp_src']}>{x['tp_dst']}{x['mode'][0]}={x['frac_of_measured_hbm']:.3f}/h{x['host_ms_per_reshard']:.2f}/d{x['ms']:.2f}" for x in r))
PY
