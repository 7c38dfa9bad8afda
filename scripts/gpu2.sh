python scripts/prof.py --calls 3 2>&1 | tail -5
python scripts/prof.py --calls 3 --no-gather 2>&1 | tail -3
ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/prof_extract -f python scripts/prof.py --calls 2 > gpurun_out/ncu1.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu1.log
