# Round evidence with the current build: smoke, GPU suite, bench (both arms), ncu launch list +
# one full capture of the bench kernel, per-config sweep, two-rank functional smoke, sanitizers.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy -s 20 -c 1 -o gpurun_out/prof_e0 \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 python scripts/configs_sweep.py > gpurun_out/configs.log 2>&1; tail -3 gpurun_out/configs.log
bash scripts/multirank_smoke.sh
bash scripts/sanitize.sh
