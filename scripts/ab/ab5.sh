timeout 1200 python -m pytest tests -m gpu -x -q -k "parity or batch" 2>&1 | tail -3
bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv_d7fe593.so paper_2504_09285_b200/libdyna_kv.so
ENGINE=3 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so
ENGINE=1 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so
