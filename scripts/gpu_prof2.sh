mkdir -p gpurun_out/so
for k in k_expand k_pack; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/${k}_$1 -f python scripts/prof.py --calls 2 > /dev/null 2>&1; echo $k rc=$?
done
cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_$1.so
