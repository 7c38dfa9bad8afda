# K2 directory kernel: C2 stage timings per directory size / occupancy variant, legacy for reference
for so in "" minb5 minb6; do
  for l in 10 11; do
    if [ -n "$so" ]; then export HGS_LIB=paper_2504_04670_b200/lib/variants/libhgs_$so.so; else unset HGS_LIB; fi
    echo "== $so lnb $l"; HGS_K2D_LNB=$l timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"
  done
done
unset HGS_LIB
echo "== legacy"; HGS_K2_LEGACY=1 timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"
