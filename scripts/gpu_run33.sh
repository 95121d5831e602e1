# compute-sanitizer memcheck on the round's new kernels (He / cumulant forcing, Esoteric Twist, AA + bounce-back)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --leak-check full --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "aa_bounce_back or esoteric or forced_collide_parity or force_model_switch or aa_equals_pull" 2>&1 | tail -6 | tee gpurun_out/sanitizer_r1b.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal_blocking_bitwise and None" 2>&1 | tail -4 | tee -a gpurun_out/sanitizer_r1b.txt
