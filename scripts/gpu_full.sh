# Full measurement session (one GPU): tests, calibration, bench, ncu, sweeps.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 1500 python scripts/calibrate.py > gpurun_out/calibrate.log 2>&1; tail -1 gpurun_out/calibrate.log
timeout 300 python bench.py --steps 1000 --warmup 10 > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for e in 0 1 3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy -s 20 -c 1 -o gpurun_out/prof_e$e \
      python bench.py --steps 20 --warmup 3 --no-cpu-baseline --engine $e > /dev/null 2>&1
done
timeout 900 python scripts/configs_sweep.py > gpurun_out/configs.log 2>&1; tail -3 gpurun_out/configs.log
timeout 300 python scripts/batch_probe.py > gpurun_out/batch_probe.log 2>&1; cat gpurun_out/batch_probe.log
timeout 1200 python scripts/overlap.py --budgets 0,32 > gpurun_out/overlap.log 2>&1; tail -8 gpurun_out/overlap.log
