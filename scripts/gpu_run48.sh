# final round-1 bench lines of every config with the final build (+ reference arm) and the
# launch list of the default bench command
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
: > gpurun_out/bench_all_r1_final.jsonl
for c in c4 c4aa c3 c3eso c3twist c2_f64 c2_f32 c5 c1; do
  steps=100; [ $c = c1 ] && steps=1000
  timeout 600 python bench.py --config $c --steps $steps --warmup 5 2>/dev/null | tail -1 >> gpurun_out/bench_all_r1_final.jsonl
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/bench_all_r1_final.jsonl
cut -c1-150 gpurun_out/bench_all_r1_final.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
grep -c k_pull gpurun_out/launches_default.csv
