# 2D temporal blocking tuned (2-3 CTAs/SM): full GPU suite, C5 / 2D SRT bench with and without
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for tb in x 0; do LBM_TEMPORAL_BLOCKING=$([ $tb = x ] && echo x || echo 0) timeout 300 python bench.py --config c5 --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-220; done
for tb in x 0; do LBM_TEMPORAL_BLOCKING=$([ $tb = x ] && echo x || echo 0) timeout 300 python bench.py --config c1 --shape 8192 8192 1 --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-220; done
timeout 300 python bench.py --config c5 --steps 100 --warmup 6 2>&1 | tail -1 > gpurun_out/bench_c5.json
