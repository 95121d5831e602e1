mkdir -p gpurun_out
python bench.py --config c4aa --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-300
python bench.py --config c3 --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-300
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "aa or config3" 2>&1 | tail -2
