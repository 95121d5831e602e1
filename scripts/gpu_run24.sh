mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -25
