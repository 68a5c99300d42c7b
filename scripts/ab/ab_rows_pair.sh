# A/B of the head-sliced kernel: one vs two items per warp in flight (DYNA_KV_ROWS_PAIR).
for i in 1 2; do
  for pair in 0 1; do
    echo "== pair=$pair"
    DYNA_KV_ROWS_PAIR=$pair timeout 300 python scripts/reshard_sweep.py --quick --out /tmp/r.json 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print(r['model'], r['tp_src'], r['tp_dst'], round(r['GBps']), round(r['frac_of_measured_hbm'],3))"
  done
done
DYNA_KV_ROWS_PAIR=1 timeout 600 python -m pytest tests/test_gpu_heads.py tests/test_ipc.py -q -x 2>&1 | tail -2
