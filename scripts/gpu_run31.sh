# He forcing + Esoteric Twist: full GPU suite, in-place pattern bench lines
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in c3twist c3eso c3; do timeout 300 python bench.py --config $c --steps 40 --warmup 4 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-260; done
