# Diagnostic (unsafe builds): which step of BULK's per-chunk accounting costs the time.
for lib in paper_2504_09285_b200/libdyna_kv.so ab_libs/libdyna_kv_diag_NO_WAIT.so ab_libs/libdyna_kv_diag_NO_PROXY.so ab_libs/libdyna_kv_diag_NO_COUNT.so; do
  echo "== $lib"
  DYNA_KV_LIB=$PWD/$lib ENGINES=2 timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
done
