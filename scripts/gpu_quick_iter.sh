# quick iteration: key parity tests + stage timings (+ optional ncu of a kernel: $1 regex, $2 tag)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or random or clustered or c1 or c2 or capacity or chunked" 2>&1 | grep -E "passed|failed|Error|assert" | head -12
timeout 300 python scripts/prof.py --calls 4 2>&1 | tail -6
if [ -n "$1" ]; then
  mkdir -p gpurun_out/so
  ncu --set full --clock-control none --import-source on -k regex:$1 -s 1 -c ${3:-1} -o gpurun_out/$2 -f python scripts/prof.py --calls 2 > gpurun_out/$2.log 2>&1; echo ncu rc=$?
  cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_$2.so
fi
