# K2 iteration on the default kernel: key parity + stage times (+ ncu when $1 given)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|Error|error"
timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|Error|error"
if [ -n "$1" ]; then
  mkdir -p gpurun_out/so
  ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/$1 -f python scripts/prof.py --calls 2 > gpurun_out/$1.log 2>&1; echo ncu rc=$?
  cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_$1.so
fi
