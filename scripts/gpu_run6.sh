mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --config c4aa --gpus 2 --steps 6 --warmup 3 --shape 256 256 64 --no-cpu 2>&1 | tail -1 | cut -c1-400
python bench.py --config c4aa --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1
