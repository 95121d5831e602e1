# full GPU suite incl. the bench contract test and the GPU TGV convergence pin
timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -6
