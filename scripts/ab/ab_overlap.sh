# A/B of the producer-coupled launch: overlap.py (c = 1024, 4096; 16 CTAs) with several builds.
for lib in "$@"; do
  echo "== $lib"
  DYNA_KV_LIB=$PWD/$lib timeout 600 python scripts/overlap.py --chunks 1024,4096 --budgets 16 --reps 3 --out /tmp/o.json 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); rc=r['ready_coupled']
        print(r['chunk'], r['sm_budget_ctas'], 'prod_alone %.1f' % r['T_prod_alone_ms'], 'chunked slow %.3f' % r['producer_slowdown'], 'ready exposed %.3f slow %.3f' % (rc['exposed_ms'], rc['producer_slowdown']))"
done
