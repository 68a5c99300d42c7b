set -x
ENGINE=0 bash scripts/ab_bench.sh ab_libs/libdyna_kv_c33ab9a.so paper_2504_09285_b200/libdyna_kv.so
ENGINE=2 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so
ENGINE=3 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so
DYNA_KV_UPLOAD_STREAM=0 ENGINE=0 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
