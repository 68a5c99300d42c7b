timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6
bash scripts/multirank_smoke.sh
timeout 300 python bench.py --steps 1000 --warmup 10 2>&1 | tail -1 > gpurun_out/bench_default.json; cat gpurun_out/bench_default.json | cut -c1-400
