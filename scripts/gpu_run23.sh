mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
