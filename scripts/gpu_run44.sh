# ncu --set full of the temporal-blocking kernels (C5 2D, C2 fp64/fp32 3D) + launch lists
mkdir -p gpurun_out
for c in c5 c2_f64 c2_f32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pull2 -s 1 -c 1 -o gpurun_out/prof_$c -f \
    python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_$c.log 2>&1
  tail -2 gpurun_out/ncu_$c.log
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 6 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
ls -la gpurun_out
