# 3D temporal blocking with prefetch (D3Q19 fp64/fp32, D3Q27 raw/SRT): full GPU suite, C2 bench with / without
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c2_f64 c2_f32; do for tb in x 0; do LBM_TEMPORAL_BLOCKING=$([ $tb = x ] && echo x || echo 0) timeout 300 python bench.py --config $c --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; done; done
timeout 300 python bench.py --config c4 --steps 100 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_c4.json; cut -c1-200 gpurun_out/bench_c4.json
