mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "temporal or forced or config2" 2>&1 | tail -4
python bench.py --config c2_f64 --steps 100 --warmup 6 --no-cpu --no-e2e --shape 1024 1024 128 2>&1 | tail -1 | cut -c1-300
LBM_TEMPORAL_BLOCKING=0 python bench.py --config c2_f64 --steps 100 --warmup 6 --no-cpu --no-e2e --shape 1024 1024 128 2>&1 | tail -1 | cut -c1-300
