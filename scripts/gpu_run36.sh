# 2D temporal blocking (k_pull2_2d): bitwise tests, C5 bench with / without
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal or resident" 2>&1 | tail -3
for tb in x 0; do LBM_TEMPORAL_BLOCKING=$([ $tb = x ] && echo x || echo 0) timeout 300 python bench.py --config c5 --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-220; done
for tb in x 0; do LBM_TEMPORAL_BLOCKING=$([ $tb = x ] && echo x || echo 0) timeout 300 python bench.py --config c1 --shape 4096 4096 1 --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-220; done
