# Item order inside a chunk: DYNA_KV_ORDER=0 (layer-major) vs 1 (block-major), vs the previous build.
for i in 1 2; do
  for cfg in "ab_libs/libdyna_kv_b796.so 0" "paper_2504_09285_b200/libdyna_kv.so 0" "paper_2504_09285_b200/libdyna_kv.so 1"; do
    set -- $cfg
    echo "== $1 order=$2"
    DYNA_KV_LIB=$PWD/$1 DYNA_KV_ORDER=$2 timeout 300 python scripts/l3_probe.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l)
        if r['cand'] in ('auto','bulk p32k st6','vec p8k u8'): print(r['rows'], r['pool_GiB'], r['tables'], r['cand'], round(r['payload_GBps']))"
    DYNA_KV_LIB=$PWD/$1 DYNA_KV_ORDER=$2 timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
  done
done
