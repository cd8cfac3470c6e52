set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
timeout 120 python scripts/profile_iter.py --steps 2 2>&1 | tail -3
PACT_SIREN_SIMT=1 timeout 120 python scripts/profile_iter.py --steps 2 2>&1 | tail -3
