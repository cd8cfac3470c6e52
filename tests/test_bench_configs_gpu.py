"""GPU parity at the benchmarked configuration (cfg3, BASELINE configs[2];
cfg4 frames are cfg3 frames) and on every cfg5-specific code path
(BASELINE configs[4]: 2048^2 @ 0.05 mm, N=1024, T=8192, K=64, P=128,
SIREN 2->256x4->1), against the reference itself (oracle/_ref, run live on
the same fp32 inputs).

  (i)   one cfg3 iteration (optimize.hpp:413-461) vs ref nf_step
  (ii)  cfg5 DAS on three 24x24 crops of the full-frame stack (beamform.hpp:77-110)
  (iii) cfg5 P=128 spectra (deconv.hpp:45-62), wavefronts on a 2048^2 SIREN
        raster (aberration.hpp:134-186) and the K=64 fused loss + dL/dw
        (optimize.hpp:234-325; the unstaged-Y Nyquist path) on sampled patches
  (iv)  one width-256 step on a cfg5 sub-grid vs ref nf_step
  (v)   the GPU simulator at cfg3 vs simulate_signals (phantom.hpp:282-362)
        on every 16th channel

Tolerances are BASELINE.json north_star's: DAS / PSF (w, H, Y) 1e-4 relative
L2; image and loss 1e-3; gradients 1e-3.
"""
from __future__ import annotations

import math
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle_lib import ref, rel_l2
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import (DeconvolveOptions, GridSpec, RingGeometry, SirenSpec,
                                       Trainer, make_patch_layout)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    r = ref()
    if r is None:
        pytest.skip("oracle/_ref/libpact_ref.so not built")
    return r


def _spec(w):
    return SirenSpec(w.hidden, w.sine_layers, w.omega0, w.out_scale, w.v0)


def _check_step(tr, st, n_patches, n_angles, tag):
    """Trainer iteration buffers vs ref nf_step outputs (pre-update values)."""
    data, tv, _ = tr.report(1)
    d_err = abs(data - st["data_term"]) / abs(st["data_term"])
    t_err = abs(tv - st["tv_term"]) / abs(st["tv_term"])
    w_err = rel_l2(tr.read(3, (n_patches, n_angles), np.float32), st["w"])
    dw_err = rel_l2(tr.read(4, (n_patches, n_angles), np.float32), st["dw"])
    g_err = rel_l2(tr.read(6, (tr.n_params,), np.float64), st["grad_theta"])
    print(f"{tag}: data {d_err:.2e} tv {t_err:.2e} w {w_err:.2e} dw {dw_err:.2e} "
          f"grad_theta {g_err:.2e}")
    assert d_err <= 1e-3 and t_err <= 1e-3
    assert w_err <= 1e-4
    assert dw_err <= 1e-3
    assert g_err <= 1e-3


# --------------------------------------------------------------------------- #
# cfg3: the benchmarked frame
# --------------------------------------------------------------------------- #

@pytest.fixture(scope="module")
def W3():
    return wl.cfg3()


@pytest.fixture(scope="module")
def sig3(ctx, W3):
    s = wl.simulate(ctx, W3, seed=0)
    torch.cuda.synchronize()
    return s


def test_cfg3_iteration_vs_reference(ctx, R, W3, sig3):
    """(i) One cfg3 iteration (seed-0 SIREN, GPU-simulated seed-0 signals):
    data / TV terms, w, dL/dw and grad theta vs the reference's step body,
    and the deconvolved image under theta_0 vs deconvolve_image."""
    w = W3
    cfg = wl.train_config(w, seed=0, epochs=1, steps_per_epoch=1)
    tr = Trainer(ctx, sig3, w.ring, w.meta, w.grid, w.mask, cfg)
    tr.step(1)
    theta = R.init_siren(0, _spec(w), tr.n_params)
    assert np.array_equal(theta, tr_theta0(ctx, w, tr.n_params))
    st = R.nf_step(sig3.double().cpu().numpy(), w.ring, w.meta, w.grid, w.mask,
                   wl.train_config(w, seed=0, workers=0), theta, want_image=True)
    lay = make_patch_layout(w.grid, w.patch_mm, w.overlap)
    assert lay.n_patches == 225
    _check_step(tr, st, lay.n_patches, w.n_angles, "cfg3 step")
    tr.close()
    # final-deconvolution path at cfg3 (deconv.hpp:176-198) under theta_0
    stack = ctx.das_stack(sig3, w.ring, w.meta, w.grid, w.v0, w.delays)
    _, dev = ctx.render_sos(_spec(w), torch.as_tensor(theta), w.grid, w.mask)
    sos_err = rel_l2(dev.double().cpu().numpy(), st["sos"] - w.v0)
    img = ctx.deconvolve_image(stack, w.delays, w.v0, dev, w.ring, w.mask, lay,
                               DeconvolveOptions(w.eps_deconv, w.n_angles, w.ray_step,
                                                 w.merge_fwhm))
    img_err = rel_l2(img.double().cpu().numpy(), st["image"])
    print(f"cfg3 SOS deviation {sos_err:.2e} image {img_err:.2e}")
    assert sos_err <= 1e-4
    assert img_err <= 1e-3


def tr_theta0(ctx, w, n):
    from paper_2409_10876_b200.api import init_siren

    th = init_siren(0, _spec(w))
    assert th.size == n
    return th


def test_cfg3_simulator_vs_reference(ctx, R, W3, sig3):
    """(v) pact_simulate_signals at cfg3 vs the reference simulator on every
    16th channel (a 32-element ring with the same angle offset has exactly
    the positions of channels 0, 16, 32, ...; core.hpp:166-173)."""
    import ctypes as C

    w = W3
    p, sos = wl.phantom_rasters(w, 0)
    g = w.grid
    sm = wl.simulation_mask(w)
    sub = RingGeometry(w.ring.n_transducers // 16, w.ring.radius, w.ring.angle_offset)
    out = np.zeros((sub.n_transducers, w.meta.n_samples))
    pr, so = np.ascontiguousarray(p), np.ascontiguousarray(sos)
    R.call("simulate_signals", g.width, g.height, g.pitch, g.origin_x, g.origin_y,
           pr.ctypes.data_as(C.c_void_p), so.ctypes.data_as(C.c_void_p), sm.center_x,
           sm.center_y, sm.radius, w.v0, sub.n_transducers, sub.radius, sub.angle_offset,
           100e-9, w.meta.dt, w.meta.t0, w.meta.n_samples, 0.05, 0, out.ctypes.data_as(C.c_void_p))
    got = sig3.double().cpu().numpy()[::16]
    err = rel_l2(got, out)
    print("cfg3 simulate (32 channels) rel L2", err)
    assert err <= 1e-4


# --------------------------------------------------------------------------- #
# cfg5 code paths
# --------------------------------------------------------------------------- #

@pytest.fixture(scope="module")
def W5():
    return wl.cfg5()


@pytest.fixture(scope="module")
def sig5(ctx, W5):
    s = wl.simulate(ctx, W5, seed=0)
    torch.cuda.synchronize()
    return s


@pytest.fixture(scope="module")
def stack5(ctx, W5, sig5):
    st = ctx.das_stack(sig5, W5.ring, W5.meta, W5.grid, W5.v0, W5.delays)
    torch.cuda.synchronize()
    return st


def _crop(grid: GridSpec, x0, y0, w, h) -> GridSpec:
    return GridSpec(w, h, grid.pitch, grid.origin_x + x0 * grid.pitch,
                    grid.origin_y + y0 * grid.pitch)


@pytest.mark.parametrize("x0,y0", [(1012, 1012), (0, 0), (2024, 700)])
def test_cfg5_das_crops(R, W5, sig5, stack5, x0, y0):
    """(ii) Three 24x24 crops (centre, a corner, the right edge) of the
    full-frame cfg5 stack vs das_stack on the crop grid (each DAS pixel is
    independent: beamform.hpp:96-108)."""
    w = W5
    c = _crop(w.grid, x0, y0, 24, 24)
    want = R.das_stack(sig5.double().cpu().numpy(), w.ring, w.meta, c, w.v0, w.delays)
    got = stack5[:, y0:y0 + 24, x0:x0 + 24].double().cpu().numpy()
    err = rel_l2(got, want)
    print(f"cfg5 DAS crop ({x0},{y0}) rel L2 {err:.2e}")
    assert err <= 1e-4


SAMPLE = (0, 15, 30, 465, 480, 500, 930, 960)  # corners, edges, centre of the 31x31 layout


def test_cfg5_spectra_wavefront_and_loss(ctx, R, W5, stack5):
    """(iii) P=128 spectra, cfg5 wavefronts and the K=64 fused loss on sampled
    patches.  At K=64, P=128 the Nyquist kernel cannot stage Y in shared
    memory (2*K*S*8 B > 200 KB), so this runs its L2 path."""
    w = W5
    lay = make_patch_layout(w.grid, w.patch_mm, w.overlap)
    P = lay.patch_pixels
    assert (P, lay.n_patches, len(w.delays)) == (128, 961, 64)
    Y = ctx.patch_spectra(lay, stack5)
    idx = torch.tensor(SAMPLE, device="cuda")
    Ys = Y.index_select(0, idx).contiguous()
    del Y
    torch.cuda.empty_cache()
    st = stack5.double().cpu().numpy()
    for k, i in enumerate(SAMPLE):
        ox, oy = (int(v) for v in lay.offsets[i])
        c = _crop(w.grid, ox, oy, P, P)
        want = R.patch_spectra(st[:, oy:oy + P, ox:ox + P], w.delays, w.v0, c, w.patch_mm,
                               w.overlap)[0]
        err = rel_l2(Ys[k].cpu().numpy(), want)
        assert err <= 1e-4, (i, err)
    # SOS: the seed-0 width-256 SIREN rendered on the 2048^2 grid
    spec = _spec(w)
    theta = R.init_siren(0, spec, spec.param_count())
    _, dev = ctx.render_sos(spec, torch.as_tensor(theta), w.grid, w.mask)
    sos = w.v0 + dev.double().cpu().numpy()
    cen = lay.centers[list(SAMPLE)]
    wf = ctx.wavefront(w.ring, w.grid, dev, w.v0, w.mask, cen, w.n_angles, w.ray_step)
    want_w = R.wavefront_profile(cen, w.ring, w.grid, sos, w.v0, w.mask, w.n_angles, w.ray_step)
    w_err = rel_l2(wf.double().cpu().numpy(), want_w)
    print(f"cfg5 wavefront rel L2 {w_err:.2e}")
    assert w_err <= 1e-4
    scale = 1.0 / (lay.n_patches * len(w.delays) * P * P)
    loss, dw = ctx.loss_grad(Ys, wf, w.delays, P, w.grid.pitch, w.eps_deconv, scale)
    loss, dw = loss.cpu().numpy(), dw.double().cpu().numpy()
    wf64 = wf.double().cpu().numpy()
    Yh = Ys.cpu().numpy()
    l_ref, dw_ref = [], []
    for k in range(len(SAMPLE)):
        lv, d = R.fused_patch_loss_grad(Yh[k], wf64[k], P, w.grid.pitch, w.n_angles, w.delays,
                                        w.eps_deconv, scale)
        l_ref.append(lv)
        dw_ref.append(d)
    l_err = rel_l2(loss, np.array(l_ref))
    dw_err = rel_l2(dw, np.array(dw_ref))
    print(f"cfg5 loss rel L2 {l_err:.2e} dw {dw_err:.2e}")
    assert l_err <= 1e-3
    assert dw_err <= 1e-3


def test_cfg5_subgrid_width256_step(ctx, R, W5, sig5):
    """(iv) One iteration with cfg5's network (2->256x4->1, streamed tcgen05
    GEMMs), K=64 delays and P=128 patches on a 256x256 sub-grid of the cfg5
    frame (9 patches) vs ref nf_step."""
    w = replace(W5, grid=GridSpec.centered(256, 256, W5.grid.pitch))
    cfg = wl.train_config(w, seed=0, epochs=1, steps_per_epoch=1)
    tr = Trainer(ctx, sig5, w.ring, w.meta, w.grid, w.mask, cfg)
    tr.step(1)
    theta = R.init_siren(0, _spec(w), tr.n_params)
    st = R.nf_step(sig5.double().cpu().numpy(), w.ring, w.meta, w.grid, w.mask,
                   wl.train_config(w, seed=0, workers=0), theta, want_image=True)
    lay = make_patch_layout(w.grid, w.patch_mm, w.overlap)
    assert (lay.patch_pixels, lay.n_patches) == (128, 9)
    _check_step(tr, st, lay.n_patches, w.n_angles, "cfg5 sub-grid step")
    tr.close()
    # the P = 128 final deconvolution (forward and inverse patch FFTs,
    # deconv.hpp:176-198) under theta_0
    stack = ctx.das_stack(sig5, w.ring, w.meta, w.grid, w.v0, w.delays)
    _, dev = ctx.render_sos(_spec(w), torch.as_tensor(theta), w.grid, w.mask)
    img = ctx.deconvolve_image(stack, w.delays, w.v0, dev, w.ring, w.mask, lay,
                               DeconvolveOptions(w.eps_deconv, w.n_angles, w.ray_step,
                                                 w.merge_fwhm))
    img_err = rel_l2(img.double().cpu().numpy(), st["image"])
    print(f"cfg5 sub-grid image (P=128) rel L2 {img_err:.2e}")
    assert img_err <= 1e-3


def test_cfg5_window_covers_lookups(W5):
    """Appendix A t0 rule: every DAS lookup of the cfg5 frame is in-window."""
    w = W5
    g = w.grid
    r_max = math.hypot((g.width - 1) * g.pitch / 2, (g.height - 1) * g.pitch / 2)
    t_min = 1e-3 * (w.ring.radius - r_max - max(w.delays)) / w.v0
    t_max = 1e-3 * (w.ring.radius + r_max - min(w.delays)) / w.v0
    assert t_min >= w.meta.t0
    assert t_max <= w.meta.t0 + (w.meta.n_samples - 1) * w.meta.dt


def test_cfg3_training_is_bitwise_deterministic(ctx, W3, sig3):
    """Two engines on the same cfg3 frame and seed give bitwise-identical
    dL/dv, gradients and parameters after two iterations: the ray adjoint
    accumulates in 64-bit fixed point (order-independent integer sums) and
    every other reduction runs in a fixed order."""
    w = W3
    cfg = wl.train_config(w, seed=0, epochs=1, steps_per_epoch=2)
    out = []
    for _ in range(2):
        tr = Trainer(ctx, sig3, w.ring, w.meta, w.grid, w.mask, cfg)
        tr.step(2)
        out.append((tr.read(5, (w.grid.height, w.grid.width), np.float64),
                    tr.read(6, (tr.n_params,), np.float64), tr.theta(), tr.report(1)))
        tr.close()
    (gv_a, g_a, th_a, r_a), (gv_b, g_b, th_b, r_b) = out
    assert np.array_equal(gv_a, gv_b)
    assert np.array_equal(g_a, g_b)
    assert np.array_equal(th_a, th_b)
    assert r_a == r_b
