for pdl in 1 0; do
  echo "PDL=$pdl"
  DYNA_KV_PDL=$pdl timeout 300 python scripts/channel_stress.py 4 4194304 1000 1 40 2>&1 | tail -4
  DYNA_KV_PDL=$pdl timeout 300 python scripts/channel_stress.py 2 1048576 100 1 40 2>&1 | tail -3
  DYNA_KV_PDL=$pdl timeout 300 python scripts/channel_stress.py 4 4194304 1000 0 40 2>&1 | tail -3
done
