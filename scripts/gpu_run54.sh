# discrete equilibrium (R29): GPU parity; full suite
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "discrete" 2>&1 | tail -5
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
