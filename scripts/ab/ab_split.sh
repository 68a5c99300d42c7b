# Signalled calls: one launch per chunk with flags released by the next launch (DYNA_KV_SIGNAL_SPLIT=1) vs VEC.
for i in 1 2; do
  for sp in 0 1; do
    printf "split=%s " $sp
    DYNA_KV_SIGNAL_SPLIT=$sp timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4), round(d['e2e']['value']))"
  done
done
DYNA_KV_SIGNAL_SPLIT=1 timeout 1200 python -m pytest tests -m gpu -q -x -rf 2>&1 | grep -vE "^\.+$" | tail -3
