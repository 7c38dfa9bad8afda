ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/prof_extract2 -f python scripts/prof.py --calls 2 > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_expand -s 1 -c 1 -o gpurun_out/prof_expand1 -f python scripts/prof.py --calls 2 > gpurun_out/ncu3.log 2>&1; echo ncu rc=$?
