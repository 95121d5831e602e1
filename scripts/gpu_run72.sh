# TB regression fix (template RANGE switch): A/B microbench, product bench, TB + peer tests
for v in d712de1 fix; do echo "== $v"; ./scripts/tb_ab_$v; done
for c in c2_f64 c2_f32 c5; do timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['metric'][:60], d['value'], d['roofline']['frac'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x -k "temporal or two_step or resident" 2>&1 | tail -2
