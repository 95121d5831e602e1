# diagnose the C5 slab-context timeout
export LBM_PEER_TIMEOUT_S=20
for r in 2 4 8; do
  echo "== ranks $r chunk 2"; timeout 300 python scripts/peer_overhead.py --config c5 --shape 8192 8192 1 --ranks $r --steps 16 --chunk 2 2>&1 | grep -v "^{" | tail -3
done
echo "== ranks 2 chunk 64"; timeout 300 python scripts/peer_overhead.py --config c5 --shape 8192 8192 1 --ranks 2 --steps 64 --chunk 64 2>&1 | grep -v "^{" | tail -3
echo "== ranks 2 chunk 64 no graphs"; LBM_CUDA_GRAPHS=0 timeout 300 python scripts/peer_overhead.py --config c5 --shape 8192 8192 1 --ranks 2 --steps 64 --chunk 64 2>&1 | grep -v "^{" | tail -3
