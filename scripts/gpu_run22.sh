mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=5
for sh in "256 256 64" "512 512 64"; do
echo "shape $sh graphs (chunk 32)"; timeout 300 python scripts/peer_overhead.py --steps 640 --ranks 2 4 --chunk 32 --shape $sh 2>&1 | head -3
echo "shape $sh eager interleaved (chunk 1)"; LBM_CUDA_GRAPHS=0 timeout 300 python scripts/peer_overhead.py --steps 640 --ranks 2 4 --chunk 1 --shape $sh 2>&1 | head -3
done
