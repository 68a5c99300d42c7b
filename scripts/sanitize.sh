# compute-sanitizer on small configs (memcheck, racecheck, synccheck); summaries in gpurun_out/sanitizer_*.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_heads.py tests/test_gpu_ready.py tests/test_gpu_batch.py \
      -q -x \
      -k "toy_config and (1000 or 17) or heads_parity and G4-G2 or heads_reblocking or cancel_before_launch or signalled_batch_per_request or signal_per_chunk_flags or batch_matches_oracle" \
      -p no:cacheprovider \
      > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitizer_$tool.log | tail -2 | tr '\n' ' ')"
done
