# A/B of the head-sliced kernel: reshard_sweep --quick with several builds, interleaved.
for i in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    DYNA_KV_LIB=$PWD/$lib timeout 300 python scripts/reshard_sweep.py --quick --out /tmp/r.json 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print(r['model'], r['tp_src'], r['tp_dst'], round(r['GBps']), round(r['frac_of_measured_hbm'],3))"
  done
done
