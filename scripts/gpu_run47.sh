# peer connect/disconnect, multi-process + slab tests, synccheck on the barrier-heavy kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -3
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_cluster_cap or (temporal_blocking_matches and None-1-1-1-1-0) or (temporal_blocking_2d and None-0-1-1-0)" 2>&1 | tail -3 | tee gpurun_out/synccheck.txt
