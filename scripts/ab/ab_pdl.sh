# PDL on/off, same library, same box.
for i in 1 2; do
  for pdl in 0 1; do
    printf "PDL=%s " $pdl
    DYNA_KV_PDL=$pdl timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4), round(d['e2e']['value']), d['config']['resolved_plan'])"
  done
done
for pdl in 0 1; do
  echo "configs PDL=$pdl"
  DYNA_KV_PDL=$pdl timeout 600 python scripts/configs_sweep.py --out gpurun_out/configs_pdl$pdl.json 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(f\"{d['config'][:70]:70s} {d['GBps']:8.1f} GB/s {d['ms']:8.3f} ms\")"
done
