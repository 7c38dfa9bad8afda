# one bench run + launch list + full ncu captures of the three main kernels
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench rc=$?
tail -2 gpurun_out/bench_r1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches rc=$?
for k in k_expand k_extract k_pack; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r1_$k -f python scripts/prof.py --calls 2 > /dev/null 2>&1; echo $k rc=$?
done
cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_r1.so
