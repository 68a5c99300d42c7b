# Item order inside a chunk (DYNA_KV_JGROUP = runs per group; 0 = layer-major): throughput, then parity with an odd group.
for J in 0 1 4 8 16 32 64 0; do
  echo "== J=$J"
  DYNA_KV_JGROUP=$J timeout 300 python scripts/l3_probe.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l)
        if r['cand'] in ('auto','bulk p32k st6','vec p8k u8','bulk_ws p32k st6'): print(r['rows'], r['pool_GiB'], r['tables'], r['cand'], round(r['payload_GBps']))" | paste -sd'|'
done
DYNA_KV_JGROUP=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_ready.py -q -x 2>&1 | tail -2
