# compute-sanitizer on small configs (memcheck, racecheck, synccheck); summaries in gpurun_out/sanitizer_*.log
# NOTE: compute-sanitizer has since been closed on this pool (runs under it left GPUs needing a reset);
# the round-1 / round-2 logs in profiles/ come from earlier boxes.  Not part of the evidence scripts.
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_heads.py tests/test_gpu_ready.py tests/test_gpu_batch.py \
      tests/test_gpu_pack.py tests/test_gpu_concurrency.py tests/test_gpu_overlap_prev.py -q -x \
      -k "toy_config and (1000 or 17) or heads_parity and G4-G2 or heads_reblocking or auto_small_rows_as_tiles and toy or batch_small_rows_as_tiles or pack_small_rows_run_as_tiles or prepared_batch_errors or cancel_before_launch or signalled_batch_per_request or signal_per_chunk_flags or batch_matches_oracle or reshard_one_launch and 2-8 or pack_unpack_host_tables or deferred_errors or interleaved_chunk_streams or ready_wait_timeout or per_chunk_calls_overlapped or batches_heads_reshard_pack_overlapped or prepared_batches_overlapped" \
      -p no:cacheprovider \
      > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitizer_$tool.log | tail -2 | tr '\n' ' ')"
done
