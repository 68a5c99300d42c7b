timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv_d7fe593.so paper_2504_09285_b200/libdyna_kv_sonf.so paper_2504_09285_b200/libdyna_kv.so
ENGINE=3 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so
