"""GPU parity of the hidden-width-128 SIREN (the tcgen05 3xTF32 layers of
csrc/siren_tc.cu, used by cfg3/cfg4) against the C oracle's restatement of
render_sos / backprop_sos (proj/include/pact/nfield.hpp:145-233).

The pixel count is deliberately not a multiple of the 128-pixel tile and the
weight-gradient split leaves ragged ranges.  Tolerances: SOS deviation 1e-5
relative L2 (the PSF budget is 1e-4), gradient 1e-3 (BASELINE north_star).
"""
import numpy as np
import pytest
import torch

from oracle_lib import orc, rel_l2
from paper_2409_10876_b200.api import CircularMask, GridSpec, SirenSpec, init_siren, masked_pixels

pytestmark = pytest.mark.gpu


def _case(width, height, layers, seed):
    grid = GridSpec(width, height, 1e-4, -0.5e-4 * width, -0.5e-4 * height)
    mask = CircularMask(0.0, 0.0, 0.45e-4 * max(width, height))
    spec = SirenSpec(128, layers, 30.0, 100.0, 1500.0)
    theta = init_siren(seed, spec)
    rng = np.random.default_rng(seed)
    theta = theta * (1.0 + 0.05 * rng.standard_normal(theta.shape))
    return grid, mask, spec, theta


@pytest.mark.parametrize("width,height,layers,seed", [(97, 83, 4, 1), (64, 64, 2, 2),
                                                      (211, 190, 3, 3)])
def test_render_sos_h128(ctx, width, height, layers, seed):
    grid, mask, spec, theta = _case(width, height, layers, seed)
    raster, dev = ctx.render_sos(spec, torch.as_tensor(theta), grid, mask)
    want = orc().render_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask)
    err = rel_l2(dev.double().cpu().numpy(), want - spec.v0)
    assert err <= 1e-5, err


@pytest.mark.parametrize("width,height,layers,seed", [(97, 83, 4, 4), (64, 64, 2, 5),
                                                      (211, 190, 3, 6)])
def test_siren_backward_h128(ctx, width, height, layers, seed):
    grid, mask, spec, theta = _case(width, height, layers, seed)
    idx, _ = masked_pixels(grid, mask)
    rng = np.random.default_rng(100 + seed)
    g = rng.standard_normal(len(idx)).astype(np.float32)
    got = ctx.siren_backward(spec, torch.as_tensor(theta), grid, mask, torch.as_tensor(g))
    want = orc().backprop_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask,
                              g.astype(np.float64))
    got = got.cpu().numpy()
    err = rel_l2(got, want)
    assert err <= 1e-3, err
    # every layer block individually (a wrong tile would hide in the global norm)
    off = 0
    for l in range(layers + 1):
        rows = 1 if l == layers else 128
        cols = 2 if l == 0 else 128
        blk = slice(off, off + rows * cols + rows)
        e = rel_l2(got[blk], want[blk])
        assert e <= 1e-3, (l, e)
        off += rows * cols + rows


def test_siren_backward_h128_many_tiles(ctx):
    """The fused per-layer backward (csrc/siren_bwd.cu) at a size where every
    CTA runs ~20 32-pixel tiles through all buffer rings (ragged last
    tile, uneven tiles per CTA), against the oracle's backprop_sos; plus the
    bias and head blocks exactly as the per-op kernels compute them."""
    grid, mask, spec, theta = _case(401, 383, 4, 9)
    idx, _ = masked_pixels(grid, mask)
    assert len(idx) % 32 != 0 and len(idx) > 148 * 32 * 4
    rng = np.random.default_rng(109)
    g = rng.standard_normal(len(idx)).astype(np.float32)
    got = ctx.siren_backward(spec, torch.as_tensor(theta), grid, mask, torch.as_tensor(g))
    want = orc().backprop_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask,
                              g.astype(np.float64))
    got = got.cpu().numpy()
    off = 0
    for l in range(spec.n_hidden_layers + 1):
        rows = 1 if l == spec.n_hidden_layers else 128
        cols = 2 if l == 0 else 128
        for blk in (slice(off, off + rows * cols), slice(off + rows * cols, off + rows * cols + rows)):
            e = rel_l2(got[blk], want[blk])
            assert e <= 1e-4, (l, e)
        off += rows * cols + rows
