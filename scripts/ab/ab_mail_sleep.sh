# Accountant poll back-off: spin (default build) vs nanosleep 256 / 2000 ns; BULK and BULK_WS with the accountant.
for i in 1 2; do
  for lib in paper_2504_09285_b200/libdyna_kv.so ab_libs/libdyna_kv_mail256.so ab_libs/libdyna_kv_mail2000.so; do
    echo "== $lib"
    DYNA_KV_LIB=$PWD/$lib DYNA_KV_ACCOUNTANT=all ENGINES=2,3 timeout 300 python scripts/sig_probe.py 2>&1 | grep '"signal": 1'
  done
done
