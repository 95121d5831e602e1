# after the RANGE fix: slab decomposition with two-step sweeps across ranks + final bench of every config
mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
for tb in 1 0; do echo "== LBM_PEER_TB=$tb"; LBM_PEER_TB=$tb timeout 300 python scripts/peer_overhead.py --config c5 --shape 8192 8192 1 --ranks 2 4 --steps 32 --chunk 2 2>&1 | grep -v "^{" | tail -3;
  LBM_PEER_TB=$tb timeout 300 python scripts/peer_overhead.py --config c2 --shape 256 256 256 --ranks 2 4 --steps 32 --chunk 2 2>&1 | grep -v "^{" | tail -3; done 2>&1 | tee gpurun_out/peer_tb_final.txt
bash scripts/gpu_run69.sh
