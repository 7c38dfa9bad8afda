ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/prof_extract4 -f python scripts/prof.py --calls 2 > gpurun_out/ncu5.log 2>&1; echo ncu rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_pack -s 1 -c 1 -o gpurun_out/prof_pack1 -f python scripts/prof.py --calls 2 > gpurun_out/ncu6.log 2>&1; echo ncu rc=$?
