# Round-2 tile-engine evidence with the final build: reshard sweeps (rows vs tiles, s = 4096 and
# 16384), configs sweep with and without tiles, ncu launch durations of whole-row TP-shard
# migrations (tiles vs VEC) and of the reshard cases.
set -x
timeout 900 python scripts/reshard_sweep.py --out gpurun_out/r02_reshard_tiles.json > /dev/null 2>&1
timeout 900 python scripts/reshard_sweep.py --s 16384 --reps 10 --out gpurun_out/r02_reshard_tiles_s16384.json > /dev/null 2>&1
timeout 900 python scripts/configs_sweep.py --out gpurun_out/r02_configs.json > /dev/null 2>&1
DYNA_KV_TILES=0 timeout 900 python scripts/configs_sweep.py --out gpurun_out/r02_configs_notiles.json > /dev/null 2>&1
for c in "llama3 8 8" "llama3 4 4" "llama3 2 2" "qwen72 8 8"; do
  for e in tiles rows; do
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_copy" --csv \
      python scripts/tiles_case.py $c --whole --engine $e --reps 3 > gpurun_out/wncu_${c// /_}_$e.csv 2>/dev/null
  done
done
for c in "llama3 1 2" "llama3 1 4" "llama3 1 8" "llama3 8 1" "llama3 4 2" "llama3 2 8" "qwen72 8 4" "qwen72 4 8" "qwen72 2 8"; do
  for e in tiles rows; do
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_copy_(tiles|rows)" --csv \
      python scripts/tiles_case.py $c --engine $e --reps 3 > gpurun_out/tncu_${c// /_}_$e.csv 2>/dev/null
  done
done
ls gpurun_out | wc -l
