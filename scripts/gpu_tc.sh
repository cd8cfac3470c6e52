timeout 300 python -m pytest tests/test_siren_tc_gpu.py -q -x 2>&1 | tail -15
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 120 python scripts/profile_iter.py --steps 2 2>&1 | tail -2
