# round-2 checkpoint: drop-in tests, bench (with C++ e2e legs), 2-rank path on one GPU, reference arm
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_parity.py -x -q -m gpu -k "dropin or hub or fallback or capacity" 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2h.json 2> gpurun_out/bench_r2h.err; echo bench rc=$?
cat gpurun_out/bench_r2h.json; tail -3 gpurun_out/bench_r2h.err
bash scripts/gpu_multirank.sh
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_r2h.json 2> gpurun_out/ref_r2h.err; echo ref rc=$?; cat gpurun_out/ref_r2h.json
