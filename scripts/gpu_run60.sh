# temporal blocking across ranks on the peer path
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -x -k "two_step" 2>&1 | tail -25
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -3
