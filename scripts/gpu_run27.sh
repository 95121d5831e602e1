mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "temporal" 2>&1 | tail -3
for c in c2_f64; do for tb in 1 0; do LBM_TEMPORAL_BLOCKING=$([ $tb = 1 ] && echo x || echo 0) python bench.py --config $c --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; done; done
python bench.py --config c2_f64 --steps 100 --warmup 6 --no-cpu --no-e2e --shape 256 256 512 2>&1 | tail -1 | cut -c1-200
LBM_TEMPORAL_BLOCKING=0 python bench.py --config c2_f64 --steps 100 --warmup 6 --no-cpu --no-e2e --shape 256 256 512 2>&1 | tail -1 | cut -c1-200
