# C5 8192^2 slab contexts on one GPU, chunk 2: temporal blocking across ranks on / off
export LBM_PEER_TIMEOUT_S=20
for tb in 1 0; do echo "== LBM_PEER_TB=$tb"; LBM_PEER_TB=$tb timeout 300 python scripts/peer_overhead.py --config c5 --shape 8192 8192 1 --ranks 2 4 --steps 32 --chunk 2 2>&1 | grep -v "^{" | tail -3; done 2>&1 | tee gpurun_out/peer_tb_c5.txt
