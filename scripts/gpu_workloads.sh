# bench lines for C1 / C3 / C4 / C5 (C2 is the default line)
for w in C1 C3 C4; do
  timeout 1200 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?
done
timeout 1500 python bench.py --workload C5 --steps 3 --warmup 1 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5 rc=$?
timeout 900 python bench.py --rng philox --steps 20 --warmup 5 --no-dropin-e2e > gpurun_out/bench_C2_philox.json 2> gpurun_out/bench_C2_philox.err; echo C2_philox rc=$?
