timeout 300 python tests/gpu_quick.py 2>&1 | grep -v "bad=\[\]" | tail -3
python scripts/prof.py --calls 3 2>&1 | tail -2 | head -1
ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/prof_extract7 -f python scripts/prof.py --calls 2 > gpurun_out/ncu9.log 2>&1; echo ncu rc=$?
