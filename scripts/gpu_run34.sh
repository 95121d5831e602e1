# cluster-resident D2Q9 loop: bitwise tests, sanitizer, C1 bench by cluster size
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "resident or config1 or graph_replay or aa_equals or bounce" 2>&1 | tail -5
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_cluster_cap" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_cluster_cap" 2>&1 | tail -3
for cap in 16 8 4 2; do LBM_RESIDENT_CLUSTER=$cap timeout 300 python bench.py --config c1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; done
LBM_RESIDENT=0 timeout 300 python bench.py --config c1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200
for s in 128 256; do timeout 300 python bench.py --config c1 --shape $s $s 1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; LBM_RESIDENT=0 timeout 300 python bench.py --config c1 --shape $s $s 1 --steps 1000 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200; done
