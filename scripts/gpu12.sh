python scripts/prof.py --calls 3 2>&1 | tail -2 | head -1
