# bench.py with and without per-step events inside the timed region (they sit between kernels).
for i in 1 2; do
  for ev in 1 0; do
    printf "step_events=%s " $ev
    DYNA_BENCH_STEP_EVENTS=$ev timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms']*1e3,1), round(d['e2e']['value']))"
  done
done
