# N = 2 bench under torchrun on one GPU (functional check of the multi-rank bench path after
# the collective PeerRunner change): peer (default) and exchange halos
for halo in auto exchange; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 10 --warmup 3 --shape 256 256 128 --halo $halo --no-cpu 2>&1 | grep '^{' | cut -c1-260
done
