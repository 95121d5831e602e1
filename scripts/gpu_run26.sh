mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "extreme or rest_state" 2>&1 | tail -15
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "graph_replay and LBM_PULL or graph_replay and 0-1-1" 2>&1 | tail -8
