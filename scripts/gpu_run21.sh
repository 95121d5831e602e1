mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -4
timeout 600 python scripts/peer_overhead.py --steps 64 --ranks 2 8 2>&1 | head -3
timeout 600 python scripts/peer_overhead.py --steps 640 --ranks 2 8 --shape 256 256 64 2>&1 | head -3
LBM_CUDA_GRAPHS=0 timeout 600 python scripts/peer_overhead.py --steps 640 --ranks 2 8 --shape 256 256 64 2>&1 | head -3
