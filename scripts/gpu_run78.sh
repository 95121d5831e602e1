# discrete CM equilibrium by closed-form binomial moments (full stencils): parity + cost
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "discrete or random_configuration" 2>&1 | tail -3
for c in c3disc c3; do timeout 300 python bench.py --config $c --steps 60 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['metric'][:100], d['value'], d['roofline']['frac'], d['config']['kernel_regs'])"; done
