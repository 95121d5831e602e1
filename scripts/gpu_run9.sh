mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
python bench.py --config c3eso --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-330
python bench.py --config c3 --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-330
python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-330
