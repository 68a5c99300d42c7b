# e2e with signalled multi-chunk calls on VEC (default) vs BULK_WS + accountant (DYNA_KV_SIGNAL_WS=1).
for i in 1 2 3; do
  for w in 0 1; do
    printf "signal_ws=%s " $w
    DYNA_KV_SIGNAL_WS=$w timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4), round(d['e2e']['value']))"
  done
done
