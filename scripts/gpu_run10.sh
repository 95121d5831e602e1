mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal or config4 or config2" 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
python bench.py --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-900
LBM_TEMPORAL_BLOCKING=0 python bench.py --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-300
python bench.py --config c2_f64 --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-300
python bench.py --config c2_f32 --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-300
