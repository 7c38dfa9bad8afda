timeout 300 python tests/gpu_quick.py 2>&1 | grep -v "bad=\[\]" | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python scripts/prof.py --calls 3 2>&1 | tail -2 | head -1
