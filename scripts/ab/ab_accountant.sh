# Signalled BULK / BULK_WS: the copying thread counts each chunk itself (default) vs an accountant thread (DYNA_KV_ACCOUNTANT=1).
for i in 1 2; do
  for a in 0 1; do
    echo "== accountant=$a"
    DYNA_KV_ACCOUNTANT=$a ENGINES=1,2,3 timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
    DYNA_KV_ACCOUNTANT=$a ENGINES=2,3 S=4096 C=512 timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
  done
done
DYNA_KV_ACCOUNTANT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "signal or litmus or fuzz_migrate" 2>&1 | tail -2
