# K1 iteration: parity files + stage times (xoshiro, then philox via prof.py)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -x -q -m gpu > gpurun_out/k1iter_tests.log 2>&1; tail -2 gpurun_out/k1iter_tests.log
for i in 1 2; do timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprof|rror"; done
timeout 300 python scripts/prof.py --calls 3 --philox 2>&1 | grep -E "call 2|unprof|rror"
