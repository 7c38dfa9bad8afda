# consumer row: GPU tests + ABI/sanitizer smoke
timeout 900 python -m pytest tests/test_gpu_consumer.py tests/test_abi.py -x -q -m gpu > gpurun_out/consumer_full.log 2>&1; tail -5 gpurun_out/consumer_full.log
grep -E "^E " gpurun_out/consumer_full.log | head -20
