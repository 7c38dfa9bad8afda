for c in 65536 16384 8192 4096 2048; do
  echo "chunk $c"; HGS_CHUNK_ROOTS=$c timeout 300 python scripts/prof.py --calls 5 2>&1 | grep unprofiled
done
