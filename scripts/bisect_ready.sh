for set in "tests/test_gpu_heads.py" "tests/test_gpu_channel.py"; do
  echo "== $set + ready"
  timeout 900 python -m pytest $set tests/test_gpu_ready.py -m gpu -q -x -o timeout=60 -k "not first_mark" 2>&1 | grep -vE "^\.+$" | tail -4
done
