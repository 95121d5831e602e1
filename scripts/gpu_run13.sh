mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5
for c in c2_f64 c2_f32; do python bench.py --config $c --steps 100 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-1100; done
python bench.py --steps 100 --warmup 6 2>&1 | tail -1 > gpurun_out/bench_c4_run13.json; cut -c1-400 gpurun_out/bench_c4_run13.json
