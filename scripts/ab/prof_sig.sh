timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_copy_bulk<.bool.1' -s 5 -c 1 -o gpurun_out/prof_bulk_sig \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --engine 2 > gpurun_out/prof_bulk_sig.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_copy_bulk<.bool.0' -s 5 -c 1 -o gpurun_out/prof_bulk_nosig \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --engine 2 > gpurun_out/prof_bulk_nosig.log 2>&1
ls -la gpurun_out/*.ncu-rep
