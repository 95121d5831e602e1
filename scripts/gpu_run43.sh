# full GPU suite after the TB prefetch change (rounding-level TB tests)
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
