# bench lines for C1 / C3 / C4 (C2 is the default line) + seed-spec test
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "seeds" 2>&1 | tail -1
for w in C1 C3 C4; do
  timeout 1200 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
  tail -c 1500 gpurun_out/bench_$w.json; echo; tail -3 gpurun_out/bench_$w.err
done
