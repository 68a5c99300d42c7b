# Tile engine round-2 evidence: full GPU suite, per-config sweep (1-GPU forms), reshard sweeps
# (rows vs tiles) at s = 4096 and 16384.
set -x
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
timeout 900 python scripts/configs_sweep.py > gpurun_out/configs.log 2>&1; cat gpurun_out/configs.log | cut -c1-220
timeout 900 python scripts/reshard_sweep.py --out gpurun_out/reshard_s4096.json > /dev/null 2>&1
timeout 900 python scripts/reshard_sweep.py --s 16384 --reps 10 --out gpurun_out/reshard_s16384.json > /dev/null 2>&1
ls gpurun_out
