# final round-1 bench lines of every config (final build) + reference arm
mkdir -p gpurun_out
: > gpurun_out/bench_all_r1_final.jsonl
for c in c4 c4aa c3 c3eso c3twist c2_f64 c2_f32 c5 c1 c4disc c3disc; do
  steps=100; [ $c = c1 ] && steps=1000
  timeout 600 python bench.py --config $c --steps $steps --warmup 5 2>/dev/null | tail -1 >> gpurun_out/bench_all_r1_final.jsonl
done
timeout 600 python bench.py --impl reference --steps 100 --warmup 5 2>/dev/null | tail -1 >> gpurun_out/bench_all_r1_final.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/bench_all_r1_final.jsonl"):
    d = json.loads(l)
    print(f"{d.get('impl','ours'):9s} {d['metric'][:90]:90s} {d['value']:10.1f} frac={d.get('roofline',{}).get('frac')} e2e={d.get('e2e',{}).get('value')}")
PY
