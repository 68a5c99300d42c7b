# Round-1 NEXT-3 evidence: head-sliced reshard throughput, layer-granular overlap, Llama-3 row probe
set -x
timeout 600 python scripts/reshard_sweep.py > gpurun_out/reshard.log 2>&1; tail -16 gpurun_out/reshard.log
timeout 900 python scripts/l3_probe.py > gpurun_out/l3_probe.log 2>&1; cat gpurun_out/l3_probe.log | cut -c1-200
timeout 600 python -m pytest tests/test_gpu_ready.py -q -x 2>&1 | tail -2
timeout 1500 python scripts/overlap.py --layers --chunks 1024,4096 --budgets 0,16 --reps 3 --out gpurun_out/overlap_layers.json > gpurun_out/overlap_layers.log 2>&1; tail -4 gpurun_out/overlap_layers.log | cut -c1-300
