# Final evidence on the round's last build: smoke, full GPU suite, bench (both arms), ncu launch list +
# one full capture of the bench kernel, configs sweep, sanitizers, fuzz x10
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_ring -s 20 -c 1 -o gpurun_out/prof_e0 \
    python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline > /dev/null 2>&1; ls gpurun_out/prof_e0*
timeout 900 python scripts/configs_sweep.py > gpurun_out/configs.log 2>&1; tail -3 gpurun_out/configs.log
DYNA_FUZZ_SCALE=10 timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/fuzz_x10.log 2>&1; tail -2 gpurun_out/fuzz_x10.log
