python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python scripts/profile_iter.py --steps 2 2>&1 | tail -2
