# one bench run + launch list + full ncu captures of the main kernels; tag = $1
tag=${1:-r1}
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench rc=$?
tail -2 gpurun_out/bench_$tag.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches rc=$?
for k in k_expand k_extract k_pack k_gather_nodes k_gather_edges_rec; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/${tag}_$k -f python scripts/prof.py --calls 2 > /dev/null 2>&1; echo $k rc=$?
done
mkdir -p gpurun_out/so; cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_$tag.so
