# Source-level ncu of the signalled BULK kernel (where does the issuing thread wait?)
timeout 900 env ENGINES=2 N=12 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -s 20 -c 2 \
   -o gpurun_out/prof_bulk_sig2 python scripts/sig_probe.py > gpurun_out/prof_bulk_sig2.log 2>&1; tail -2 gpurun_out/prof_bulk_sig2.log
S=4096 C=512 timeout 600 python scripts/sig_probe.py 2>&1 | tail -6
