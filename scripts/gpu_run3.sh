mkdir -p gpurun_out
./scripts/variants 2>&1 | tee gpurun_out/variants.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q --durations=10 2>&1 | tail -15
