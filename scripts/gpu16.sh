ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/prof_extract9 -f python scripts/prof.py --calls 2 > /dev/null 2>&1; echo ncu rc=$?
