"""GPU parity of the hidden-width-256 SIREN (cfg5's 2 -> 256 x 4 -> 1) on the
streamed tcgen05 3xTF32 GEMMs of csrc/siren_wide.cu, against the C oracle's
restatement of render_sos / backprop_sos (proj/include/pact/nfield.hpp:145-233).

Pixel counts are not multiples of the 128-pixel tile or the 32-pixel
weight-gradient chunk.  Tolerances as for width 128: SOS deviation 1e-5
relative L2 (PSF budget 1e-4), every gradient block 1e-3 (north_star).
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
    spec = SirenSpec(256, layers, 30.0, 100.0, 1500.0)
    theta = init_siren(seed, spec)
    rng = np.random.default_rng(seed)
    theta = theta * (1.0 + 0.05 * rng.standard_normal(theta.shape))
    return grid, mask, spec, theta


@pytest.mark.parametrize("width,height,layers,seed", [(97, 83, 4, 11), (150, 139, 2, 12)])
def test_render_sos_h256(ctx, width, height, layers, seed):
    grid, mask, spec, theta = _case(width, height, layers, seed)
    _, dev = ctx.render_sos(spec, torch.as_tensor(theta), grid, mask)
    want = orc().render_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask)
    err = rel_l2(dev.double().cpu().numpy(), want - spec.v0)
    assert err <= 1e-5, err


@pytest.mark.parametrize("width,height,layers,seed", [(97, 83, 4, 13), (150, 139, 3, 14)])
def test_siren_backward_h256(ctx, width, height, layers, seed):
    grid, mask, spec, theta = _case(width, height, layers, seed)
    idx, _ = masked_pixels(grid, mask)
    rng = np.random.default_rng(100 + seed)
    g = rng.standard_normal(len(idx)).astype(np.float32)
    got = ctx.siren_backward(spec, torch.as_tensor(theta), grid, mask, torch.as_tensor(g))
    want = orc().backprop_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask,
                              g.astype(np.float64))
    got = got.cpu().numpy()
    off = 0
    for l in range(layers + 1):
        rows = 1 if l == layers else 256
        cols = 2 if l == 0 else 256
        for blk in (slice(off, off + rows * cols), slice(off + rows * cols, off + rows * cols + rows)):
            e = rel_l2(got[blk], want[blk])
            assert e <= 1e-3, (l, e)
        off += rows * cols + rows


@pytest.mark.parametrize("hidden", [128, 256])
@pytest.mark.parametrize("width,height,layers", [(13, 11, 2), (13, 11, 4), (7, 5, 3)])
def test_siren_tiny_masks(ctx, hidden, width, height, layers):
    """Masks smaller than one tile (fewer pixels than a 32- or 128-pixel tile,
    a single CTA or a single 2-CTA cluster with an empty partner tile): the
    tensor-core paths still match the oracle and terminate."""
    grid = GridSpec(width, height, 1e-4, -0.5e-4 * width, -0.5e-4 * height)
    mask = CircularMask(0.0, 0.0, 0.45e-4 * max(width, height))
    spec = SirenSpec(hidden, layers, 30.0, 100.0, 1500.0)
    theta = init_siren(7, spec)
    idx, _ = masked_pixels(grid, mask)
    assert 0 < len(idx) < 128
    _, dev = ctx.render_sos(spec, torch.as_tensor(theta), grid, mask)
    want = orc().render_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask)
    assert rel_l2(dev.double().cpu().numpy(), want - spec.v0) <= 1e-5
    g = np.random.default_rng(3).standard_normal(len(idx)).astype(np.float32)
    got = ctx.siren_backward(spec, torch.as_tensor(theta), grid, mask, torch.as_tensor(g)).cpu().numpy()
    want = orc().backprop_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask,
                              g.astype(np.float64))
    assert rel_l2(got, want) <= 1e-3
