# cluster-resident D2Q9 loop: start-of-kernel cluster barrier, eligibility rule; tests + sanitizers + C1 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "resident or config1 or graph_replay or aa_equals or bounce" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident" 2>&1 | tail -3 | tee gpurun_out/sanitizer_resident.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_cluster_cap" 2>&1 | tail -12 | tee -a gpurun_out/sanitizer_resident.txt
timeout 300 python bench.py --config c1 --steps 1000 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_c1.json; cut -c1-300 gpurun_out/bench_c1.json
