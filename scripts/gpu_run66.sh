# full GPU suite after temporal blocking across ranks
timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -3
