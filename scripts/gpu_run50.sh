# resident loop with an H-deep halo: bitwise tests, sanitizers, C1 bench per halo depth
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "resident or smallest or config1" 2>&1 | tail -3
LBM_RESIDENT_HALO=4 timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_cluster_cap" 2>&1 | tail -2 | tee gpurun_out/sanitizer_halo.txt
LBM_RESIDENT_HALO=4 timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_cluster_cap" 2>&1 | tail -2 | tee -a gpurun_out/sanitizer_halo.txt
LBM_RESIDENT_HALO=4 timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_halo and 64" 2>&1 | tail -2 | tee -a gpurun_out/sanitizer_halo.txt
for h in 1 2 3 4; do LBM_RESIDENT_HALO=$h timeout 300 python bench.py --config c1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-140; done
for h in 1 2; do LBM_RESIDENT_HALO=$h timeout 300 python bench.py --config c1 --shape 128 128 1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-140; done
for h in 1 2 3 4; do LBM_RESIDENT_CLUSTER=8 LBM_RESIDENT_HALO=$h timeout 300 python bench.py --config c1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-140; done
