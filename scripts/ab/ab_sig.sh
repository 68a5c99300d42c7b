# A/B of per-chunk signalling cost per engine (scripts/sig_probe.py) across builds, interleaved.
for i in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    DYNA_KV_LIB=$PWD/$lib timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
  done
done
