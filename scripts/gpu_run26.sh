mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "extreme or rest_state" 2>&1 | tail -3
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "cuda_graph_replay" 2>&1 | tail -5 | tee gpurun_out/sanitizer_graphs.txt
