bash scripts/ab_overlap.sh paper_2504_09285_b200/libdyna_kv.so ab_libs/libdyna_kv_e0f5b63.so
timeout 600 python -m pytest tests/test_gpu_ready.py -q -x 2>&1 | tail -2
