# Evidence for the head-sliced kernel and the new control paths: IPC reshard test, sanitizers, one ncu capture.
set -x
timeout 600 python -m pytest tests/test_ipc.py -q -x 2>&1 | tail -2
bash scripts/sanitize.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_rows -s 6 -c 1 -o gpurun_out/prof_rows \
    python scripts/reshard_sweep.py --quick --reps 2 --out /tmp/r.json > gpurun_out/prof_rows.log 2>&1; tail -3 gpurun_out/prof_rows.log
