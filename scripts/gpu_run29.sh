# cumulant body force (R26): GPU parity + Poiseuille + temporal-blocking bitwise
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "force or temporal or poiseuille" 2>&1 | tail -4
