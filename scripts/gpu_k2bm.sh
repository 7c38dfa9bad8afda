# K2 bitmap-directory kernel: parity + timing (+ variants, + ncu)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu -k "c2_full or c4 or alternative or fuzz" 2>&1 | tail -3
echo "== hash"; HGS_K2=hash timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled|Error|error"
for so in paper_2504_04670_b200/lib/libhgs.so paper_2504_04670_b200/lib/variants/*.so; do
  echo "== $so"; HGS_LIB=$so timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled|Error|error"
done
mkdir -p gpurun_out/so
ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/k2_bm -f python scripts/prof.py --calls 2 > gpurun_out/k2_bm.log 2>&1; echo ncu rc=$?
cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_k2_bm.so
