mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15
python scripts/dam_break.py --out gpurun_out/dam_break.json 2>&1 | tail -5
./scripts/layout_copy 2>&1 | tee gpurun_out/layout_copy.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --shape 256 256 64 --no-cpu 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck --leak-check full python -m pytest tests/test_gpu_parity.py -q -x -k "aa_equals_pull or bounce_back or init_and_macroscopic or check_finite" 2>&1 | tail -6
timeout 600 compute-sanitizer --tool initcheck python -m pytest tests/test_gpu_parity.py -q -x -k "test_config3 or test_diagnostics" 2>&1 | tail -6
python bench.py --steps 100 --warmup 5 > gpurun_out/bench_c4_run5.json 2>&1; tail -1 gpurun_out/bench_c4_run5.json
