timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
ENGINE=2 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so paper_2504_09285_b200/libdyna_kv_prev.so
