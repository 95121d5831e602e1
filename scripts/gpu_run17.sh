mkdir -p gpurun_out
export LBM_PEER_TIMEOUT_S=20
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6
python bench.py --steps 50 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_c4_run17.json; cut -c1-300 gpurun_out/bench_c4_run17.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
