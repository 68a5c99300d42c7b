set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "round_trip" 2>&1 | tail -2
timeout 1500 python scripts/overlap.py --budgets 0,4,16 --chunks 512,1024,4096 > gpurun_out/overlap.log 2>&1; tail -3 gpurun_out/overlap.log
