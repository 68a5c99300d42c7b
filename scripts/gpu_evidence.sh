# Round evidence with the current build: smoke, GPU suite, bench (both arms), ncu launch list of the
# bench + one full capture of the bench kernel, per-config sweep, multi-rank functional smoke,
# sanitizers, native latency probe, overlap (P:738 analogue).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_ring -s 20 -c 1 -o gpurun_out/prof_e0 \
    python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline > /dev/null 2>&1; ls gpurun_out/prof_e0*
timeout 900 python scripts/configs_sweep.py > gpurun_out/configs.log 2>&1; tail -3 gpurun_out/configs.log
nvcc -O2 -o /tmp/latency_probe scripts/native/latency_probe.c -I include -L paper_2504_09285_b200 -ldyna_kv \
    -Xlinker -rpath=$PWD/paper_2504_09285_b200 && timeout 300 /tmp/latency_probe > gpurun_out/latency_probe.jsonl; cat gpurun_out/latency_probe.jsonl
timeout 1500 python scripts/overlap.py --chunks 512,1024,4096 --budgets 0,16 --layers --out gpurun_out/overlap.json 2>&1 | tail -4
