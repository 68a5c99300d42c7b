# ncu --set full captures of the round-2 kernels (one launch each, after warm-up), pulled back
# as .ncu-rep; summaries are written on the CPU box with scripts/ncu_summary.py.
set -x
for w in c2 t4 rows small; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_ -s 2 -c 1 \
      -o gpurun_out/prof_r02_$w python scripts/ncu_step.py --work $w > gpurun_out/prof_r02_$w.log 2>&1
  tail -2 gpurun_out/prof_r02_$w.log
done
ls -la gpurun_out/*.ncu-rep
