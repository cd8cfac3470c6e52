# Fused SIREN backward: parity tests, stage times fused vs per-op kernels.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_siren_tc_gpu.py -q -x 2>&1 | tail -15
timeout 300 python scripts/profile_iter.py --steps 2 2>&1 | tail -3
PACT_SIREN_FUSED_BWD=0 timeout 300 python scripts/profile_iter.py --steps 2 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
