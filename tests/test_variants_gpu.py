"""A/B parity of the round-2b kernels against the variants they replaced, on
one cfg3 iteration (the benchmarked frame), each variant in its own process
(the switches are read once per process; scripts/dump_step.py):

  * the interior ray adjoint as a cell gather vs the per-ray kernel
    (PACT_RAY_CELLS=0): dL/dv, the gradient and dL/dw;
  * the adjoint's border-line steps as a per-border-cell gather vs the
    per-ray items (PACT_RAY_SIDE=0): dL/dv and the gradient;
  * the SIREN forward on split-fp16 MMAs with two tiles in flight vs 3xTF32
    (PACT_SIREN_F16=0): the wavefronts, dL/dv and the gradient;
  * the SIREN backward on split-fp16 MMAs (power-of-two operand scales) vs
    3xTF32 (PACT_SIREN_BWD_F16=0): the gradient (the forward is identical).

Both products are fp32-accurate: the cell gather sums the same deposits in
another order (fixed point per cell corner), split fp16 carries the same 22
significant bits as the TF32 split.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _step(tmp_path, name, env):
    out = tmp_path / f"{name}.npz"
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "dump_step.py"), str(out)],
                   check=True, env=e, cwd=ROOT, timeout=600)
    return np.load(out)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.gpu
def test_cell_gather_and_f16_chain_vs_replaced_variants(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    prod = _step(tmp_path, "product", {})
    cells_off = _step(tmp_path, "cells_off", {"PACT_RAY_CELLS": "0"})
    tf32 = _step(tmp_path, "tf32", {"PACT_SIREN_F16": "0"})
    side_off = _step(tmp_path, "side_off", {"PACT_RAY_SIDE": "0"})
    # side gather vs per-ray border-line items: same forward, adjoint to fixed-point rounding
    assert np.array_equal(prod["w"], side_off["w"])
    e_gv, e_g = _rel(prod["gv"], side_off["gv"]), _rel(prod["grad"], side_off["grad"])
    print(f"side gather vs per-ray: dL/dv {e_gv:.2e} grad {e_g:.2e}")
    assert e_gv <= 1e-6 and e_g <= 1e-6  # (a run's fp32 pixel sums group steps differently)
    # cell gather vs per-ray adjoint: same forward, adjoint to fixed-point rounding
    assert np.array_equal(prod["w"], cells_off["w"])
    e_gv, e_g = _rel(prod["gv"], cells_off["gv"]), _rel(prod["grad"], cells_off["grad"])
    print(f"cell gather vs per-ray: dL/dv {e_gv:.2e} grad {e_g:.2e}")
    assert e_gv <= 1e-6 and e_g <= 1e-6  # (corner sums from the cell's four fp32 moments)
    # split-fp16 chain vs 3xTF32 chain
    e_w, e_gv2, e_g2 = (_rel(prod[k], tf32[k]) for k in ("w", "gv", "grad"))
    print(f"split fp16 vs 3xTF32 forward: w {e_w:.2e} dL/dv {e_gv2:.2e} grad {e_g2:.2e}")
    assert e_w <= 1e-5 and e_gv2 <= 1e-5 and e_g2 <= 1e-5
    # split-fp16 backward vs 3xTF32 backward: same forward and adjoint
    bwd32 = _step(tmp_path, "bwd_tf32", {"PACT_SIREN_BWD_F16": "0"})
    assert np.array_equal(prod["w"], bwd32["w"]) and np.array_equal(prod["gv"], bwd32["gv"])
    e_g3 = _rel(prod["grad"], bwd32["grad"])
    print(f"split fp16 vs 3xTF32 backward: grad {e_g3:.2e}")
    assert e_g3 <= 1e-5
    # closed-form run sums vs step sums in the border-cell gather
    steps = _step(tmp_path, "side_steps", {"PACT_SIDE_SERIES": "0"})
    e_w4, e_gv4, e_g4 = (_rel(prod[k], steps[k]) for k in ("w", "gv", "grad"))
    print(f"run series vs step sums: w {e_w4:.2e} dL/dv {e_gv4:.2e} grad {e_g4:.2e}")
    assert e_w4 <= 1e-6 and e_gv4 <= 1e-5 and e_g4 <= 1e-5
