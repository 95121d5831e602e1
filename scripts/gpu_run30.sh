# He forcing (R27) + cumulant forcing (R26): GPU parity
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "force or temporal or poiseuille" 2>&1 | tail -4
