for cfg in "--engine 1 --unroll 8 --piece 8192" "--engine 1 --unroll 16 --piece 16384" "--engine 1 --unroll 16 --piece 32768" "--engine 1 --unroll 4 --piece 4096" "--engine 0"; do
  printf "%s: " "$cfg"
  timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), d['config']['resolved_plan'])"
done
