# A/B: the same bench on the same box with two builds of the library (interleaved).
for i in 1 2; do
  for lib in paper_2504_09285_b200/libdyna_kv.so paper_2504_09285_b200/libdyna_kv_ab.so; do
    echo "== $lib"
    DYNA_KV_LIB=$PWD/$lib timeout 300 python bench.py --steps 1000 --warmup 10 --engine 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'])"
  done
done
