mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python scripts/table3_roundoff.py --steps 200000 --every 2000 --out gpurun_out/table3_roundoff.json 2>&1 | tee gpurun_out/table3.txt
