timeout 300 python tests/gpu_quick.py 2>&1 | grep -v "bad=\[\]" | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python scripts/prof.py --calls 3 2>&1 | tail -2 | head -1
ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/prof_extract6 -f python scripts/prof.py --calls 2 > gpurun_out/ncu8.log 2>&1; echo ncu rc=$?
