mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 300 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -2
timeout 600 python scripts/peer_overhead.py --steps 30 --ranks 2 4 8 2>&1 | head -4
