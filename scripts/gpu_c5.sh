timeout 1500 python bench.py --workload C5 --steps 3 --warmup 1 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5 rc=$?
cat gpurun_out/bench_C5.json; tail -3 gpurun_out/bench_C5.err
