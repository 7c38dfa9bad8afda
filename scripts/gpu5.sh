timeout 300 python tests/gpu_quick.py 2>&1 | grep -v "bad=\[\]" | tail -8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python scripts/prof.py --calls 3 2>&1 | tail -2
HGS_HASH_SLOTS_PER_KEY=2 python scripts/prof.py --calls 3 2>&1 | tail -2
HGS_HASH_SLOTS_PER_KEY=8 python scripts/prof.py --calls 3 2>&1 | tail -2
python scripts/prof.py --calls 3 --philox 2>&1 | tail -2
