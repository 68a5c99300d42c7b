# Final-build refresh of the overlap, reshard and latency evidence.
set -x
timeout 2400 python scripts/overlap.py --layers --chunks 512,1024,2048,4096 --budgets 0,32,16 --reps 3 \
    --out gpurun_out/overlap_final.json > gpurun_out/overlap_final.log 2>&1; tail -2 gpurun_out/overlap_final.log | cut -c1-200
timeout 600 python scripts/reshard_sweep.py --out gpurun_out/reshard_final.json > gpurun_out/reshard_final.log 2>&1; tail -3 gpurun_out/reshard_final.log
nvcc -O2 -Wno-deprecated-gpu-targets -o /tmp/latency_probe scripts/native/latency_probe.c -I include -L paper_2504_09285_b200 \
    -ldyna_kv -Xlinker -rpath=$PWD/paper_2504_09285_b200 && timeout 600 /tmp/latency_probe > gpurun_out/latency_final.jsonl; tail -2 gpurun_out/latency_final.jsonl
