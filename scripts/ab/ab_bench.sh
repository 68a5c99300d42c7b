# A/B: the same bench on the same box with several builds of the library (interleaved).
# usage: bash scripts/ab_bench.sh lib1.so lib2.so ...   (default: current vs libdyna_kv_ab.so)
LIBS="$@"
[ -z "$LIBS" ] && LIBS="paper_2504_09285_b200/libdyna_kv.so paper_2504_09285_b200/libdyna_kv_ab.so"
for i in 1 2; do
  for lib in $LIBS; do
    printf "%s " "$lib"
    DYNA_KV_LIB=$PWD/$lib timeout 300 python bench.py --steps 1000 --warmup 10 --engine ${ENGINE:-2} --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4), round(d['e2e']['value']), d['config']['resolved_plan'])"
  done
done
