# TMA tile engine for head slices: parity (heads + reshard + fuzz), reshard sweep rows vs tiles, racecheck.
set -x
timeout 900 python -m pytest tests/test_gpu_heads.py -q -x -p no:cacheprovider > gpurun_out/tiles_tests.log 2>&1; tail -3 gpurun_out/tiles_tests.log
timeout 900 python scripts/reshard_sweep.py --out gpurun_out/reshard_tiles.json > gpurun_out/reshard_tiles.log 2>&1; tail -40 gpurun_out/reshard_tiles.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_heads.py tests/test_gpu_parity.py -q -x -p no:cacheprovider \
   -k "heads_parity and G4-G2 and tiles or reshard_one_launch and 2-8 or toy_config and 1000" > gpurun_out/tiles_racecheck.log 2>&1; grep -E 'RACECHECK SUMMARY|passed|failed|Race' gpurun_out/tiles_racecheck.log | head
