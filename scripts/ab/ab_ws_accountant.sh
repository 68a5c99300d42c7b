# BULK_WS signalling: storer counts itself (default) vs an accountant warp (DYNA_KV_WS_ACCOUNTANT=1).
for i in 1 2; do
  for a in 0 1; do
    echo "== accountant=$a"
    DYNA_KV_WS_ACCOUNTANT=$a ENGINES=1,3 timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
    DYNA_KV_WS_ACCOUNTANT=$a ENGINES=3 S=4096 C=512 timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
  done
done
DYNA_KV_WS_ACCOUNTANT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "signal or litmus" 2>&1 | tail -2
