# ncu of the head-slice kernels on one reshard launch (s = 16384): launch durations for every quick
# case and engine, and one --set full capture each of the tile kernel on Llama-3-8B 1->8 and 8->1.
set -x
for c in "llama3 1 4" "llama3 1 8" "llama3 8 1" "llama3 4 2" "qwen72 8 4" "qwen72 4 8"; do
  for e in tiles rows; do
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_copy_(tiles|rows)" --csv \
      python scripts/tiles_case.py $c --engine $e --reps 3 > gpurun_out/tncu_${c// /_}_$e.csv 2>/dev/null
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_tiles -s 2 -c 1 -o gpurun_out/prof_tiles_1to8 python scripts/tiles_case.py llama3 1 8 --reps 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_tiles -s 2 -c 1 -o gpurun_out/prof_tiles_8to1 python scripts/tiles_case.py llama3 8 1 --reps 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_tiles -s 2 -c 1 -o gpurun_out/prof_tiles_q8to4 python scripts/tiles_case.py qwen72 8 4 --reps 3 > /dev/null 2>&1
ls gpurun_out/
