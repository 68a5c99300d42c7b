# Where the signalled ring's cost goes (unsafe diagnostic builds drop one step each), and the
# interleaved reshard with plans staged in shared memory.
set -x
python -m pytest tests/test_gpu_heads.py -q -x -p no:cacheprovider -k "reshard" 2>&1 | tail -2
python scripts/reshard_sweep.py --quick --out gpurun_out/reshard_r02d.json 2>&1 | cut -c1-200 | tail -12
W="--work c2batch,t4prime --cand plain=0:0:0:0:0 --cand sig=0:0:0:0:0:1"
AB_TAG=sig_full python scripts/engine_ab.py $W 2>&1 | tail -4
DYNA_KV_ACCOUNTANT=0 AB_TAG=sig_noacc python scripts/engine_ab.py $W 2>&1 | tail -4
for d in NO_WAIT NO_PROXY NO_COUNT; do DYNA_KV_LIB=ab_libs/libdyna_kv_diag_$d.so AB_TAG=sig_$d python scripts/engine_ab.py $W 2>&1 | tail -4; done
