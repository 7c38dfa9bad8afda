# K2 v2 (bucket sort, leaner scan): parity then timing
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 300 python scripts/prof.py --calls 4 2>&1 | tail -3
