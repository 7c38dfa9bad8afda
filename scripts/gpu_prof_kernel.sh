# usage: bash scripts/gpu_prof_kernel.sh <kernel-regex> <tag> [prof.py args]
k=$1; tag=$2; shift 2
mkdir -p gpurun_out/so
timeout 300 python scripts/prof.py --calls 3 "$@" 2>&1 | tail -2 | head -1
ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/$tag -f python scripts/prof.py --calls 2 "$@" > gpurun_out/$tag.log 2>&1; echo ncu rc=$?
cp paper_2504_04670_b200/lib/libhgs.so gpurun_out/so/libhgs_$tag.so
