# compute-sanitizer on the peer two-step path (memcheck; racecheck of the shared-memory ring)
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_slabs.py -q -x -k "two_step" 2>&1 | tail -3 | tee gpurun_out/sanitizer_peer_tb.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_slabs.py -q -x -k "two_step and 0-1-1-1" 2>&1 | tail -3 | tee -a gpurun_out/sanitizer_peer_tb.txt
