for c in 65536 32768 16384 8192; do
  echo "chunk $c"; HGS_CHUNK_ROOTS=$c timeout 300 python scripts/prof.py --calls 5 2>&1 | grep unprofiled
done
