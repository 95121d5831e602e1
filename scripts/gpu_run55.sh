# cost of the discrete equilibrium (R29) on the HBM-bound D3Q27 kernels
for c in c4disc c4 c3disc c3; do timeout 300 python bench.py --config $c --steps 60 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['metric'][:100], d['value'], d['roofline']['frac'], d['config']['kernel_regs'])"; done
