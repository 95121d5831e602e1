mkdir -p gpurun_out
for c in c3 c4aa c3eso; do python bench.py --config $c --steps 50 --warmup 6 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-250; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "aa or config3 or esoteric" 2>&1 | tail -2
