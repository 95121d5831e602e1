mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 600 python scripts/peer_overhead.py --steps 30 --ranks 2 4 8 2>&1 | tee gpurun_out/peer_overhead.txt
