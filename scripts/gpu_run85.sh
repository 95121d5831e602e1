# exchange-path two-step regions: in-process + torchrun multi-process + slab/peer regressions
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_multiprocess.py -q -x 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 scripts/slab_check.py --steps 9 --halo exchange 2>&1 | grep -E "TB|ALL"
