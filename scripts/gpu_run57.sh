# final build: full GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench_default_final.json; cut -c1-200 gpurun_out/bench_default_final.json
