# K1 decision-parallel xoshiro: parity tests, then C2 stage timings (group GL=4 default, GL=2, GL=8, serial)
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu -k "c2_full or c3 or fuzz" 2>&1 | tail -2
echo "== group GL4"; timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"
for v in k1x2 k1x8; do echo "== $v"; HGS_LIB=paper_2504_04670_b200/lib/variants/libhgs_$v.so timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"; done
echo "== serial"; HGS_K1_SERIAL=1 timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"
echo "== philox"; timeout 300 python scripts/prof.py --calls 3 --philox 2>&1 | grep -E "call 2|unprofiled"
