timeout 300 python tests/gpu_quick.py 2>&1 | grep -v "bad=\[\]" | tail -4
for spk in 2 3 4; do HGS_HASH_SLOTS_PER_KEY=$spk python scripts/prof.py --calls 3 2>&1 | tail -2 | head -1; done
