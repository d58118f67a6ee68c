python -m pytest tests/test_distributed.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/shard_tests.log 2>&1; echo rc=$? >> gpurun_out/shard_tests.log
tail -5 gpurun_out/shard_tests.log
python tools/shard_probe.py 2 1 2 4 8 > gpurun_out/shard_probe.log 2>&1
python tools/shard_probe.py 3 8 >> gpurun_out/shard_probe.log 2>&1
cat gpurun_out/shard_probe.log
