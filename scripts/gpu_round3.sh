set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python scripts/ready_probe.py 2>&1 | tail -9
for e in 0 1; do timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --engine $e 2>&1 | tail -1 | cut -c1-250; done
timeout 1500 python scripts/overlap.py --budgets 0,32 > gpurun_out/overlap.log 2>&1; tail -8 gpurun_out/overlap.log
