# Reshard with the by-value slice geometry; signalled ring: stores committed after a chunk switch
# before its bytes are counted (DYNA_BULK_DEFER 2 / 4 (default) / 8 / 16).
set -x
python -m pytest tests/test_gpu_heads.py -q -x -p no:cacheprovider 2>&1 | tail -2
python scripts/reshard_sweep.py --out gpurun_out/reshard_r02c.json 2>&1 | cut -c1-200 | tail -30
W="--work c2batch,t4prime --cand plain=0:0:0:0:0 --cand sig=0:0:0:0:0:1"
AB_TAG=defer4 python scripts/engine_ab.py $W 2>&1 | tail -4
for d in 2 8 16; do DYNA_KV_LIB=ab_libs/libdyna_kv_defer$d.so AB_TAG=defer$d python scripts/engine_ab.py $W 2>&1 | tail -4; done
AB_TAG=defer4b python scripts/engine_ab.py $W 2>&1 | tail -4
