# VEC engine compiled for 4 resident CTAs per SM (64 regs, small spills) vs 3 (80 regs).
for i in 1 2; do
  for lib in paper_2504_09285_b200/libdyna_kv.so ab_libs/libdyna_kv_vec4.so; do
    echo "== $lib"
    DYNA_KV_LIB=$PWD/$lib ENGINES=1 timeout 300 python scripts/sig_probe.py 2>&1 | grep engine
  done
done
bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so ab_libs/libdyna_kv_vec4.so
