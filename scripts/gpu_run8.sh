mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8
python bench.py --steps 100 --warmup 5 --no-cpu 2>&1 | tail -1 | cut -c1-700
