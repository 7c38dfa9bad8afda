timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "seeds or epoch" 2>&1 | tail -3
for w in C3 C5; do
  timeout 1500 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
  head -c 1200 gpurun_out/bench_$w.json; echo; tail -3 gpurun_out/bench_$w.err
done
