"""GPU parity of part 1 (das_stack, beamform.hpp:77-110) through the C-ABI.

Tolerance (BASELINE.json north_star): relative L2 <= 1e-4 against the fp64
reference on the same fp32-rounded signals.  Known-answer tests follow
proj/tests/test_beamform.cpp with fp32-appropriate margins.
"""
import numpy as np
import pytest
import torch

import golden_util as gu
from oracle_lib import orc, rel_l2
from paper_2409_10876_b200 import _abi
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import GridSpec, RingGeometry, SignalMetaInfo

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _gpu_das(ctx, sig, ring, meta, grid, v0, delays):
    s = torch.as_tensor(np.ascontiguousarray(sig, dtype=np.float32)).cuda()
    out = ctx.das_stack(s, ring, meta, grid, v0, list(delays))
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


@pytest.mark.parametrize("name", ["das_edge", "das_cfg1_crop"])
def test_das_stack_matches_reference_golden(ctx, name):
    z = gu.load(name)
    got = _gpu_das(ctx, z["sig"], gu.ring(z["ring"]), gu.meta(z["meta"]), gu.grid(z["grid"]),
                   float(z["v0"]), z["delays"])
    assert rel_l2(got, z["out"]) <= TOL


def test_das_stack_cfg1_full_vs_oracle(ctx):
    w = wl.cfg1()
    sig = wl.iid_signals(w, 0)
    got = _gpu_das(ctx, sig, w.ring, w.meta, w.grid, w.v0, w.delays)
    want = orc().das_stack(sig.astype(np.float64), w.ring, w.meta, w.grid, w.v0, w.delays)
    err = rel_l2(got, want)
    print("cfg1 DAS rel L2", err)
    assert err <= TOL


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
def test_das_stack_full_size_crop_vs_oracle(ctx, cfg):
    """Full-size GPU stack; the oracle evaluates a 24x24 crop (a sub-GridSpec
    with the same pixel positions gives identical values in the reference)."""
    w = wl.CONFIGS[cfg]()
    rng = np.random.default_rng(7)
    sig = rng.standard_normal((w.ring.n_transducers, w.meta.n_samples)).astype(np.float32)
    got = _gpu_das(ctx, sig, w.ring, w.meta, w.grid, w.v0, w.delays)
    g = w.grid
    for (x0, y0) in [(0, 0), (g.width // 2 - 12, g.height // 3), (g.width - 24, g.height - 24)]:
        crop = GridSpec(24, 24, g.pitch, g.origin_x + x0 * g.pitch, g.origin_y + y0 * g.pitch)
        want = orc().das_stack(sig.astype(np.float64), w.ring, w.meta, crop, w.v0, w.delays)
        assert rel_l2(got[:, y0:y0 + 24, x0:x0 + 24], want) <= TOL


def test_das_stack_elements_equal_das_bitwise(ctx):
    # test_beamform.cpp:99-111: das_stack[j] == das(d_j)
    w = wl.cfg1()
    sig = torch.as_tensor(wl.iid_signals(w, 3)).cuda()
    g = GridSpec.centered(33, 33, 0.1)
    delays = [-0.4, 0.0, 0.3]
    st = ctx.das_stack(sig, w.ring, w.meta, g, 1500.0, delays)
    for j, d in enumerate(delays):
        single = ctx.das(sig, w.ring, w.meta, g, 1500.0, d)
        assert torch.equal(st[j], single)


def test_zero_signals_give_zero_image(ctx):
    w = wl.cfg1()
    sig = torch.zeros((w.ring.n_transducers, w.meta.n_samples), device="cuda")
    out = ctx.das_stack(sig, w.ring, w.meta, w.grid, w.v0, w.delays)
    assert torch.count_nonzero(out).item() == 0


def test_das_is_linear_in_the_signals(ctx):
    # test_beamform.cpp:79-97 (fp32 margin)
    w = wl.cfg1()
    rng = np.random.default_rng(9)
    s1 = rng.standard_normal((128, 1024)).astype(np.float32)
    s2 = (rng.uniform(-1, 1, (128, 1024)) * 1e3).astype(np.float32)
    a, b = 0.7, -1.3
    mix = (a * s1.astype(np.float64) + b * s2.astype(np.float64)).astype(np.float32)
    g = GridSpec.centered(17, 17, 0.1)
    ia = _gpu_das(ctx, s1, w.ring, w.meta, g, 1500.0, [0.0])
    ib = _gpu_das(ctx, s2, w.ring, w.meta, g, 1500.0, [0.0])
    im = _gpu_das(ctx, mix, w.ring, w.meta, g, 1500.0, [0.0])
    scale = max(np.abs(ia).max(), np.abs(ib).max())
    assert np.abs(im - (a * ia + b * ib)).max() <= 1e-5 * scale


def _point_source_signals(ring, meta, v0=1500.0, sigma=100e-9, src=(0.0, 0.0)):
    # simulate_signals (phantom.hpp:340-361) for one point source, uniform SOS
    pos = ring.positions()
    t = meta.t0 + np.arange(meta.n_samples) * meta.dt
    out = np.zeros((ring.n_transducers, meta.n_samples))
    for n in range(ring.n_transducers):
        tau = 1e-3 * np.hypot(pos[n, 0] - src[0], pos[n, 1] - src[1]) / v0
        u = (t - tau) / sigma
        v = (2.0 / sigma) * (1 - u * u) * np.exp(-0.5 * u * u)
        v[np.abs(t - tau) > 6 * sigma] = 0
        out[n] = v
    return out.astype(np.float32)


def test_das_focuses_centered_point_and_delay_gives_ring(ctx):
    # test_beamform.cpp:55-70
    ring = RingGeometry(128, 50.0, 0.0)
    meta = SignalMetaInfo(1400, 25e-9, 32.0e-6, 1500.0)
    sig = _point_source_signals(ring, meta)
    g = GridSpec.centered(65, 65, 0.1)
    img = _gpu_das(ctx, sig, ring, meta, g, 1500.0, [0.0])[0]
    by, bx = np.unravel_index(np.argmax(np.abs(img)), img.shape)
    assert (bx, by) == (32, 32)
    img = _gpu_das(ctx, sig, ring, meta, g, 1500.0, [0.5])[0]
    by, bx = np.unravel_index(np.argmax(np.abs(img)), img.shape)
    r = np.hypot(*g.world(bx, by))
    assert 0.35 < r < 0.65


def test_one_pitch_delay_shift_is_one_pixel_shift(ctx):
    # test_beamform.cpp:113-131 (fp32 margin instead of 1e-9)
    ring = RingGeometry(3, 50.0, 0.0)
    meta = SignalMetaInfo(400, 25e-9, 2.8e-5, 1500.0)
    sig = np.zeros((3, 400), np.float32)
    sig[0, 200] = 1.0
    g = GridSpec.centered(65, 65, 0.1)
    y0 = _gpu_das(ctx, sig, ring, meta, g, 1500.0, [0.2])[0]
    y1 = _gpu_das(ctx, sig, ring, meta, g, 1500.0, [0.3])[0]
    row = 32
    np.testing.assert_allclose(y1[row, :-1], y0[row, 1:], atol=2e-5)


def test_validation_errors_match_reference(ctx):
    w = wl.cfg1()
    sig = torch.zeros((128, 1024), device="cuda")
    with pytest.raises(_abi.ValidationError, match="strictly increasing"):
        ctx.das_stack(sig, w.ring, w.meta, w.grid, 1500.0, [0.1, 0.1])
    with pytest.raises(_abi.ValidationError, match="v0 must be > 0"):
        ctx.das_stack(sig, w.ring, w.meta, w.grid, -1.0, [0.0])


def test_context_launches_on_torchs_current_stream(ctx):
    """No explicit synchronize: torch's D2H copy must observe the kernel."""
    w = wl.cfg1()
    sig = torch.as_tensor(wl.iid_signals(w, 5)).cuda()
    a = ctx.das_stack(sig, w.ring, w.meta, w.grid, w.v0, w.delays).cpu()
    s2 = torch.stack([sig, sig]).sum(0) * 0.5  # same values, new buffer
    b = ctx.das_stack(s2, w.ring, w.meta, w.grid, w.v0, w.delays).cpu()
    assert torch.equal(a, b) and a.abs().max() > 0
