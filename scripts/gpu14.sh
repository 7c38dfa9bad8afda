timeout 300 python tests/gpu_quick.py 2>&1 | grep -c "bad=\[\]"
timeout 300 python tests/gpu_quick.py 2>&1 | grep "bad=\['" | head -3
python scripts/prof.py --calls 3 2>&1 | tail -2 | head -1
