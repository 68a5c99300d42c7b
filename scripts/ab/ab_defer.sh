ENGINE=2 bash scripts/ab_bench.sh paper_2504_09285_b200/libdyna_kv.so paper_2504_09285_b200/libdyna_kv_d16.so
