# one ncu --set full capture of K1 (k_expand) at C2 + the .so it ran (tag = $1)
mkdir -p gpurun_out/so
ncu --set full --clock-control none --import-source on -k regex:k_expand -s 1 -c 1 -o gpurun_out/$1 -f python scripts/prof.py --calls 2 > gpurun_out/$1.log 2>&1; echo ncu rc=$?
cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_$1.so
