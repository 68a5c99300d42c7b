# Round-2 bench session: GPU tests touched this round, the N = 1 bench (both arms), the
# multi-rank functional smoke, and the ncu launch list of the bench command.
set -x
python -m pytest tests/test_gpu_batch.py tests/test_gpu_pack.py tests/test_gpu_concurrency.py -q -p no:cacheprovider 2>&1 | tail -8
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 3000 gpurun_out/bench_n1.json; tail -5 gpurun_out/bench_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -c 800 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
