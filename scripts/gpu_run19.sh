mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 300 python -m pytest tests/test_gpu_slabs.py -q -x 2>&1 | tail -2
for f in 1 0; do echo "LBM_PEER_FENCE=$f"; LBM_PEER_FENCE=$f timeout 600 python scripts/peer_overhead.py --steps 30 --ranks 2 4 8 2>&1 | head -4; done
