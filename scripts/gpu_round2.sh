set -x
timeout 300 python scripts/ready_probe.py 2>&1 | tail -12
bash scripts/multirank_smoke.sh
bash scripts/ab_pdl.sh
