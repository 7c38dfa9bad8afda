# quick K2 iteration: key parity (with HGS_K2=$K2) + timing of hash and the selected kernel (+ ncu when $1 given)
export HGS_K2=${K2:-bm}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or random or clustered or hub or big" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu -k "c2_full or alternative" 2>&1 | tail -2
for k in hash $HGS_K2; do
  echo "== $k"; HGS_K2=$k timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled|Error|error"
done
if [ -n "$1" ]; then
  mkdir -p gpurun_out/so
  ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/$1 -f python scripts/prof.py --calls 2 > gpurun_out/$1.log 2>&1; echo ncu rc=$?
  cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_$1.so
fi
