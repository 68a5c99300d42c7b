# DYNA_MIGRATE_OVERLAP_PREV: tests + launch-bubble probe (default, flag, flag + signal, diagnostic no-wait build)
set -x
timeout 1200 python -m pytest tests/test_gpu_overlap_prev.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_heads.py tests/test_gpu_concurrency.py tests/test_gpu_ready.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > gpurun_out/ovp_tests.log 2>&1; tail -5 gpurun_out/ovp_tests.log
python scripts/ab/pdl_nowait_probe.py > gpurun_out/ovp_probe.jsonl 2>&1
DYNA_PROBE_OV=1 python scripts/ab/pdl_nowait_probe.py >> gpurun_out/ovp_probe.jsonl 2>&1
DYNA_PROBE_SIG=1 python scripts/ab/pdl_nowait_probe.py >> gpurun_out/ovp_probe.jsonl 2>&1
DYNA_PROBE_OV=1 DYNA_PROBE_SIG=1 python scripts/ab/pdl_nowait_probe.py >> gpurun_out/ovp_probe.jsonl 2>&1
DYNA_KV_LIB=$PWD/abtmp/libdyna_kv_nowait.so python scripts/ab/pdl_nowait_probe.py >> gpurun_out/ovp_probe.jsonl 2>&1
cat gpurun_out/ovp_probe.jsonl
