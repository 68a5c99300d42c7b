timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "DYNA_|^E  |passed|failed|FAILED" | head -20
timeout 1800 python scripts/calibrate.py > gpurun_out/calibrate.log 2>&1; tail -1 gpurun_out/calibrate.log
bash scripts/sanitize.sh
