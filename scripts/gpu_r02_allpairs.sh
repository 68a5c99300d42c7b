# configs[4] all pairs emulated on one GPU: GPU test + measurement (world 8 and 4)
set -x
timeout 900 python -m pytest tests/test_gpu_allpairs.py tests/test_gpu_channel.py -q -p no:cacheprovider > gpurun_out/allpairs_test.log 2>&1; tail -3 gpurun_out/allpairs_test.log
timeout 900 python scripts/allpairs_one_gpu.py --world 8 > gpurun_out/allpairs_w8.json 2> gpurun_out/allpairs_w8.err; cat gpurun_out/allpairs_w8.json; tail -3 gpurun_out/allpairs_w8.err
timeout 600 python scripts/allpairs_one_gpu.py --world 4 > gpurun_out/allpairs_w4.json 2> gpurun_out/allpairs_w4.err; cat gpurun_out/allpairs_w4.json
timeout 900 python scripts/allpairs_one_gpu.py --world 8 --mode per-receiver > gpurun_out/allpairs_w8_per.json 2>&1; cat gpurun_out/allpairs_w8_per.json
