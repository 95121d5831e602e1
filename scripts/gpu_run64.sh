# diagnose: C5-like 8 slab contexts on one GPU
export LBM_PEER_TIMEOUT_S=15
for shape in "1024 1024 1" "2048 2048 1" "8192 2048 1"; do
  echo "== c5 $shape ranks 8 chunk 2"; LBM_PEER_TB=0 timeout 200 python scripts/peer_overhead.py --config c5 --shape $shape --ranks 8 --steps 8 --chunk 2 2>&1 | grep -v "^{" | tail -2
done
echo "== c5 8192^2 ranks 8 chunk 1 no graphs"; LBM_CUDA_GRAPHS=0 LBM_PEER_TB=0 timeout 200 python scripts/peer_overhead.py --config c5 --shape 8192 8192 1 --ranks 8 --steps 4 --chunk 1 2>&1 | grep -v "^{" | tail -2
echo "== c4 ranks 8"; timeout 300 python scripts/peer_overhead.py --config c4 --ranks 8 --steps 8 --chunk 2 2>&1 | grep -v "^{" | tail -2
