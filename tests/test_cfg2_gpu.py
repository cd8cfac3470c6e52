"""GPU parity at BASELINE configs[1] (cfg2: N=256, T=2048, 256x256 @0.1 mm,
K=16, 49 patches of 64x64, SIREN 2->64x3->1) against the reference itself
(tests/golden/cfg2_step.npz: simulated signals, one forward + gradient
evaluation at the seed-0 SIREN and the deconvolved image, all through
oracle/_ref).  Tolerances as in BASELINE.json north_star."""
import numpy as np
import pytest
import torch

import golden_util as gu
from oracle_lib import rel_l2
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import (DeconvolveOptions, SirenSpec, Trainer, make_patch_layout)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    return gu.load("cfg2_step")


@pytest.fixture(scope="module")
def W():
    return wl.cfg2()


@pytest.fixture(scope="module")
def stack(ctx, G, W):
    sig = torch.as_tensor(G["sig"]).cuda()
    return ctx.das_stack(sig, W.ring, W.meta, W.grid, W.v0, W.delays)


def test_das_stack_crop(G, W, stack):
    c = gu.grid(G["crop"])
    x0 = round((c.origin_x - W.grid.origin_x) / W.grid.pitch)
    y0 = round((c.origin_y - W.grid.origin_y) / W.grid.pitch)
    got = stack[:, y0:y0 + 32, x0:x0 + 32].double().cpu().numpy()
    assert rel_l2(got, G["das_crop"]) <= 1e-4


def _spec(W):
    return SirenSpec(W.hidden, W.sine_layers, W.omega0, W.out_scale, W.v0)


def test_render_sos(ctx, G, W):
    _, dev = ctx.render_sos(_spec(W), torch.as_tensor(G["theta"]), W.grid, W.mask)
    assert rel_l2(dev.double().cpu().numpy(), G["sos"].astype(np.float64) - W.v0) <= 1e-4


def test_psf_wavefront_and_transfer(ctx, G, W):
    lay = make_patch_layout(W.grid, W.patch_mm, W.overlap)
    dev = torch.as_tensor((G["sos"].astype(np.float64) - W.v0).astype(np.float32)).cuda()
    w = ctx.wavefront(W.ring, W.grid, dev, W.v0, W.mask, lay.centers, W.n_angles, W.ray_step)
    assert rel_l2(w.double().cpu().numpy(), G["w"]) <= 1e-4
    H = ctx.transfer_stack(torch.as_tensor(G["w"][24:25].astype(np.float32)).cuda(), W.delays, 64,
                           W.grid.pitch)[0]
    assert rel_l2(H.cpu().numpy(), G["H24"]) <= 1e-4


def test_iteration_loss_and_gradient(ctx, G, W):
    cfg = wl.train_config(W, seed=0, epochs=1, steps_per_epoch=1)
    sig = torch.as_tensor(G["sig"]).cuda()
    tr = Trainer(ctx, sig, W.ring, W.meta, W.grid, W.mask, cfg)
    tr.step(1)
    data, tv, total = tr.report(1)
    assert abs(data - float(G["data_term"])) <= 1e-3 * abs(float(G["data_term"]))
    assert abs(tv - float(G["tv_term"])) <= 1e-3 * abs(float(G["tv_term"]))
    n = 49
    w = tr.read(3, (n, W.n_angles), np.float32)
    assert rel_l2(w, G["w"]) <= 1e-4
    dw = tr.read(4, (n, W.n_angles), np.float32)
    assert rel_l2(dw, G["dw"]) <= 1e-3
    g = tr.read(6, (tr.n_params,), np.float64)
    err = rel_l2(g, G["grad_theta"])
    print("cfg2 grad rel L2", err)
    assert err <= 1e-3
    tr.close()


def test_deconvolved_image(ctx, G, W, stack):
    _, dev = ctx.render_sos(_spec(W), torch.as_tensor(G["theta"]), W.grid, W.mask)
    lay = make_patch_layout(W.grid, W.patch_mm, W.overlap)
    img = ctx.deconvolve_image(stack, W.delays, W.v0, dev, W.ring, W.mask, lay,
                               DeconvolveOptions(W.eps_deconv, W.n_angles, W.ray_step, W.merge_fwhm))
    err = rel_l2(img.double().cpu().numpy(), G["image"])
    print("cfg2 image rel L2", err)
    assert err <= 1e-3


def test_simulated_signals_match_reference_simulator(ctx, G, W):
    """pact_simulate_signals (phantom.hpp:282-362) vs the reference's own
    simulate_signals on the same seeded phantom (how the fixture was made)."""
    sig = wl.simulate(ctx, W, seed=0)
    err = rel_l2(sig.double().cpu().numpy(), G["sig"].astype(np.float64))
    print("cfg2 simulate rel L2", err)
    assert err <= 1e-4


@pytest.mark.parametrize("hidden,fixture", [(128, "cfg2_h128_step"), (256, "cfg2_h256_step")])
def test_iteration_wide_network(ctx, G, W, hidden, fixture):
    """cfg2's geometry and signals with cfg3's network (SIREN 2 -> 128 x 4 -> 1:
    the fused tcgen05 forward of siren_chain.cu and the fused per-layer
    backward of siren_bwd.cu) or cfg5's (2 -> 256 x 4 -> 1: the streamed
    tcgen05 GEMMs of siren_wide.cu) inside the training step's CUDA graph;
    reference values from tests/golden/<fixture>.npz (one nf_step of
    oracle/_ref)."""
    from dataclasses import replace

    H = gu.load(fixture)
    w = replace(W, hidden=hidden, sine_layers=4)
    cfg = wl.train_config(w, seed=0, epochs=1, steps_per_epoch=1)
    tr = Trainer(ctx, torch.as_tensor(G["sig"]).cuda(), w.ring, w.meta, w.grid, w.mask, cfg)
    tr.step(1)
    data, tv, _ = tr.report(1)
    assert abs(data - float(H["data_term"])) <= 1e-3 * abs(float(H["data_term"]))
    assert abs(tv - float(H["tv_term"])) <= 1e-3 * abs(float(H["tv_term"]))
    n = 49
    assert rel_l2(tr.read(3, (n, w.n_angles), np.float32), H["w"]) <= 1e-4
    assert rel_l2(tr.read(4, (n, w.n_angles), np.float32), H["dw"]) <= 1e-3
    g = tr.read(6, (tr.n_params,), np.float64)
    err = rel_l2(g, H["grad_theta"])
    print(f"cfg2 / H={hidden} grad rel L2", err)
    assert err <= 1e-3
    tr.close()


def test_border_runs_on_a_rough_field(ctx, W):
    """The closed-form border-line runs (raymarch.cu: forward items and the
    border-cell gather) near their validity limit and past it.  cfg2's ring
    (60 mm) lies outside its 25.6 mm grid, so every ray ends in the
    border-line regime.  A field with jumps of up to ~25 % between
    neighbouring pixels makes |u| n exceed 0.2 on the long runs (those are
    summed step by step) and leaves the others with |u k| ~ 0.1, where the
    dropped u^6 term is ~1e-6.  Wavefront and adjoint of nine patches against
    the oracle (aberration.hpp:134-186, 333-361)."""
    from oracle_lib import orc

    lay = make_patch_layout(W.grid, W.patch_mm, W.overlap)
    cen = np.asarray(lay.centers).reshape(-1, 2)[::6][:9].copy()
    rng = np.random.default_rng(11)
    Hh, Ww = W.grid.height, W.grid.width
    dev = torch.as_tensor(rng.uniform(-180.0, 180.0, (Hh, Ww)).astype(np.float32)).cuda()
    sos32 = W.v0 + dev.double().cpu().numpy()
    w = ctx.wavefront(W.ring, W.grid, dev, W.v0, W.mask, cen, W.n_angles, W.ray_step)
    want_w = orc().wavefront_profile(cen, W.ring, W.grid, sos32, W.v0, W.mask, W.n_angles,
                                     W.ray_step)
    e_w = rel_l2(w.double().cpu().numpy(), want_w)
    dw32 = rng.standard_normal(want_w.shape).astype(np.float32)
    gv = ctx.ray_backward(W.ring, W.grid, dev, W.v0, W.mask, cen, W.n_angles, W.ray_step,
                          torch.as_tensor(dw32).cuda())
    want_g = np.zeros((Hh, Ww))
    for p, c in enumerate(cen):
        want_g = orc().wavefront_grad_trace(c, W.ring, W.grid, sos32, W.v0, W.mask, W.n_angles,
                                            W.ray_step, dw32[p].astype(np.float64), want_g)
    e_g = rel_l2(gv.cpu().numpy().reshape(Hh, Ww), want_g)
    print(f"rough field: w {e_w:.2e} dL/dv {e_g:.2e}")
    assert e_w <= 1e-5 and e_g <= 1e-5

