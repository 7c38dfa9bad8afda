timeout 300 python tests/gpu_quick.py 2>&1 | grep -v "bad=\[\]" | tail -20
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python scripts/prof.py --calls 3 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
tail -3 gpurun_out/bench2.err
