# final-build ncu --set full of the C4 stream-collide kernel (512^2 x 128 lattice, as in run 5)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pull -s 2 -c 1 -o gpurun_out/prof_c4_final -f \
  python bench.py --config c4 --shape 512 512 128 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_final.log 2>&1
tail -2 gpurun_out/ncu_c4_final.log
