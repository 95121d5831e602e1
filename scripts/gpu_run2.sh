mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
for c in c3 c2_f64 c2_f32 c5 c1; do python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pull -s 3 -c 1 -o gpurun_out/prof_c4 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --shape 512 512 128 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
