# fused K3: parity subset, then stage timings fused vs unfused
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "feature_widths or golden or c1 or c2 or random or capacity or chunked or hub" 2>&1 | tail -3
echo "== fused"; timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"
echo "== unfused"; HGS_K3_FUSED=0 timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"
for u in 2 8; do echo "== fused U$u"; HGS_LIB=paper_2504_04670_b200/lib/variants/libhgs_k3u$u.so timeout 300 python scripts/prof.py --calls 3 2>&1 | grep -E "call 2|unprofiled"; done
