# round-2 refresh: full GPU suite, smoke, bench + launch list, workloads, reference arm, ncu summaries
bash scripts/gpu_full.sh r2b 1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_r2b.json 2> gpurun_out/ref_r2b.err; echo ref rc=$?; cat gpurun_out/ref_r2b.json
for w in C1 C3 C4 C5; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dropin-e2e > gpurun_out/bench_r2b_$w.json 2> gpurun_out/bench_r2b_$w.err; echo $w rc=$?; done
timeout 600 python bench.py --rng philox --steps 10 --warmup 3 --no-cpu-baseline --no-dropin-e2e > gpurun_out/bench_r2b_C2_philox.json 2> gpurun_out/bench_r2b_C2_philox.err; echo philox rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_extract|k_expand|k_pack|k_gather" -c 5 -o gpurun_out/r2b_kernels -f python scripts/prof.py --calls 1 > gpurun_out/r2b_kernels.log 2>&1; echo ncu rc=$?
mkdir -p gpurun_out/so; cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_r2b.so
