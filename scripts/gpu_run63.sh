# slab decomposition on one GPU with / without temporal blocking across ranks (C5 8192^2, C2 256^3)
mkdir -p gpurun_out
for tb in 1 0; do
  echo "== LBM_PEER_TB=$tb"
  LBM_PEER_TB=$tb timeout 600 python scripts/peer_overhead.py --config c5 --shape 8192 8192 1 --ranks 2 4 8 --steps 64 2>&1 | grep -v "^{"
  LBM_PEER_TB=$tb timeout 600 python scripts/peer_overhead.py --config c2 --shape 256 256 256 --ranks 2 4 --steps 64 2>&1 | grep -v "^{"
  LBM_PEER_TB=$tb timeout 600 python scripts/peer_overhead.py --config c4 --ranks 2 4 --steps 30 2>&1 | grep -v "^{"
done 2>&1 | tee gpurun_out/peer_tb.txt
