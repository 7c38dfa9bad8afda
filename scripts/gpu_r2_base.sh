# round-2 baseline: full GPU suite, smoke, bench, launch list, one ncu --set full of k_extract
bash scripts/gpu_full.sh r2a 1
bash scripts/gpu_ncu_k2.sh
timeout 600 python scripts/prof.py --calls 4 2>&1 | tail -8
