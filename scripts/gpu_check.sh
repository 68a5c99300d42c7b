# GPU-box check: smoke, GPU tests, bench lines, optional ncu / overlap / calibration runs.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
if [ -z "$NOTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} 2>&1 | tail -30; fi
if [ -n "$CALIB" ]; then timeout 1500 python scripts/calibrate.py > gpurun_out/calibrate.log 2>&1; tail -2 gpurun_out/calibrate.log; fi
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
  for e in 0 1; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy -s 20 -c 2 -o gpurun_out/prof_e$e \
        python bench.py --steps 20 --warmup 3 --no-cpu-baseline --engine $e > gpurun_out/ncu_full_e$e.log 2>&1
  done
fi
if [ -z "$NOBENCH" ]; then
  for e in 1 2; do timeout 300 python bench.py --steps 1000 --warmup 10 --engine $e --no-cpu-baseline 2>&1 | tail -1; done
  timeout 300 python bench.py --steps 1000 --warmup 10 2>&1 | tail -1 > gpurun_out/bench_default.json; cat gpurun_out/bench_default.json
fi
if [ -n "$OVERLAP" ]; then timeout 900 python scripts/overlap.py > gpurun_out/overlap.log 2>&1; tail -20 gpurun_out/overlap.log; fi
if [ -n "$CONFIGS" ]; then timeout 900 python scripts/configs_sweep.py > gpurun_out/configs.log 2>&1; tail -20 gpurun_out/configs.log; fi
if [ -n "$PROBE" ]; then
  timeout 300 python scripts/batch_probe.py 2>&1 | tail -8
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy -s 3 -c 1 -o gpurun_out/prof_batch_bulk \
      env ONLY=batch-bulk-2 python scripts/batch_probe.py > gpurun_out/ncu_batch.log 2>&1
fi
