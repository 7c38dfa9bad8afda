# one full ncu capture of k_extract (C2) for per-line instruction/stall shares
mkdir -p gpurun_out/so
ncu --set full --clock-control none --import-source on -k regex:k_extract -s 1 -c 1 -o gpurun_out/k2_base -f python scripts/prof.py --calls 2 > gpurun_out/k2_base.log 2>&1; echo ncu rc=$?
cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_k2_base.so
