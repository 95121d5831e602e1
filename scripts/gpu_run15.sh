mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "graph or aa_equals or config1 or temporal or esoteric" 2>&1 | tail -4
for c in c1; do python bench.py --config $c --steps 1000 --warmup 5 --no-cpu 2>&1 | tail -1 | cut -c1-1500; done
LBM_CUDA_GRAPHS=0 python bench.py --config c1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-300
for s in "128 128 1" "256 256 1" "512 512 1" "1024 1024 1"; do for gr in 1 0; do LBM_CUDA_GRAPHS=$gr python bench.py --config c1 --shape $s --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; done; done
for s in "32 32 32" "64 64 64"; do for gr in 1 0; do LBM_CUDA_GRAPHS=$gr python bench.py --config c4 --shape $s --steps 640 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; done; done
