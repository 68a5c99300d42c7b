ENGINE=2 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so paper_2504_09285_b200/libdyna_kv_fenced.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_sig.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --engine 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launches_sig.csv')) if len(r)>10]
h=rows[0]; i=h.index('Kernel Name'); v=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]: agg[r[i][:60]].append(float(r[v].replace(',',''))/1000)
for k,x in agg.items(): print(f"{k:60s} n={len(x)} mean={sum(x)/len(x):.1f} us")
PY
