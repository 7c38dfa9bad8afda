timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or random or c1" 2>&1 | tail -2
python scripts/prof.py --calls 3 2>&1 | tail -2 | head -1
