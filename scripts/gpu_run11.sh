mkdir -p gpurun_out
./scripts/tb_variants 2>&1 | tee gpurun_out/tb_variants.txt
ncu --set full --clock-control none --import-source on -k regex:k_pull2 -s 2 -c 1 -o gpurun_out/prof_pull2 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --shape 512 512 128 > gpurun_out/ncu_pull2.log 2>&1
tail -2 gpurun_out/ncu_pull2.log
