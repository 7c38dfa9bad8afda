for so in paper_2504_04670_b200/lib/libhgs.so paper_2504_04670_b200/lib/variants/*.so; do
  echo "== $so"
  HGS_LIB=$so timeout 300 python scripts/prof.py --calls 3 --philox 2>&1 | grep -E "call 2|unprofiled" | sed "s/SampleCounts.*kernel ms//"
done
