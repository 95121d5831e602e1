mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 600 python -m pytest tests/test_gpu_slabs.py -q -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -30
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --shape 256 256 128 --no-e2e 2>&1 | tail -3 | cut -c1-1500
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 20 --warmup 3 --shape 256 256 128 --no-e2e --halo exchange 2>&1 | tail -3 | cut -c1-600
