"""GPU parity of parts 2 and 3 on the reference's SmallInstance fixture
(proj/tests/test_support.hpp:38-75) against outputs of the reference itself
(tests/golden/small_instance.npz, generated through oracle/_ref).

Tolerances (BASELINE.json north_star): PSF (H) and wavefront within 1e-4
relative L2; deconvolved image and loss within 1e-3; gradients within 1e-3.
"""
import numpy as np
import pytest
import torch

import golden_util as gu
from oracle_lib import rel_l2
from paper_2409_10876_b200.api import (DeconvolveOptions, SirenSpec, Trainer, joint_reconstruct,
                                       make_patch_layout, masked_pixels)
from dataclasses import replace

pytestmark = pytest.mark.gpu

PSF_TOL = 1e-4
IMG_TOL = 1e-3
LOSS_TOL = 1e-3
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def G():
    return gu.load("small_instance")


@pytest.fixture(scope="module")
def si():
    return gu.small_instance()


def _meta(G):
    return gu.meta(G["meta"])


def _dev(G):
    return torch.as_tensor((G["sos"] - 1500.0).astype(np.float32)).cuda()


def test_das_stack(ctx, G, si):
    sig = torch.as_tensor(G["sig"]).cuda()
    st = ctx.das_stack(sig, si.ring, _meta(G), si.grid, 1500.0, si.cfg.delays)
    assert rel_l2(st.double().cpu().numpy(), G["stack"]) <= 1e-4


def test_render_sos(ctx, G, si):
    cfg = si.cfg
    spec = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, 1500.0)
    raster, dev = ctx.render_sos(spec, torch.as_tensor(G["theta2"]), si.grid, si.mask)
    err = rel_l2(dev.double().cpu().numpy(), G["sos"] - 1500.0)
    assert err <= 1e-5, err
    assert rel_l2(raster.double().cpu().numpy(), G["sos"]) <= 1e-7


def test_wavefront_profile(ctx, G, si):
    lay = make_patch_layout(si.grid, si.cfg.patch_mm, si.cfg.overlap)
    w = ctx.wavefront(si.ring, si.grid, _dev(G), 1500.0, si.mask, lay.centers, si.cfg.n_angles,
                      si.cfg.ray_step)
    err = rel_l2(w.double().cpu().numpy(), G["w"])
    assert err <= PSF_TOL, err


def test_transfer_stack(ctx, G, si):
    w = torch.as_tensor(G["w"][:1].astype(np.float32)).cuda()
    H = ctx.transfer_stack(w, si.cfg.delays, 32, si.grid.pitch)[0]
    err = rel_l2(H.cpu().numpy(), G["H0"])
    assert err <= PSF_TOL, err


def test_patch_spectra(ctx, G, si):
    lay = make_patch_layout(si.grid, si.cfg.patch_mm, si.cfg.overlap)
    stack = torch.as_tensor(G["stack"].astype(np.float32)).cuda()
    Y = ctx.patch_spectra(lay, stack)
    err = rel_l2(Y.cpu().numpy(), G["Y"])
    assert err <= 1e-5, err


def test_fused_loss_and_dw(ctx, G, si):
    cfg = si.cfg
    n, K = G["Y"].shape[:2]
    scale = 1.0 / (n * K * 32 * 32)
    Y = torch.as_tensor(G["Y"]).cuda()
    w = torch.as_tensor(G["w"].astype(np.float32)).cuda()
    loss, dw = ctx.loss_grad(Y, w, cfg.delays, 32, si.grid.pitch, cfg.eps_deconv, scale, True)
    assert rel_l2(loss.cpu().numpy(), G["loss_patch"]) <= LOSS_TOL
    err = rel_l2(dw.double().cpu().numpy(), G["dw"])
    assert err <= GRAD_TOL, err


def test_ray_backward(ctx, G, si):
    cfg = si.cfg
    lay = make_patch_layout(si.grid, cfg.patch_mm, cfg.overlap)
    dw = torch.as_tensor(G["dw"].astype(np.float32)).cuda()
    gv = ctx.ray_backward(si.ring, si.grid, _dev(G), 1500.0, si.mask, lay.centers, cfg.n_angles,
                          cfg.ray_step, dw)
    idx, _ = masked_pixels(si.grid, si.mask)
    got = gv.cpu().numpy().ravel()[idx]
    want = G["grad_v_masked"] - G["tv_grad"]
    err = rel_l2(got, want)
    assert err <= GRAD_TOL, err


def tv_unambiguous(grid, mask, sos, rtol=1e-6):
    """Masked pixels none of whose TV pairs has |dv| below fp32 resolution
    (sign() there is a tie in one precision and not the other)."""
    idx, _ = masked_pixels(grid, mask)
    W, H = grid.width, grid.height
    inm = np.zeros(W * H, bool)
    inm[idx] = True
    v = sos.ravel()
    amb = np.zeros(W * H, bool)
    for p in idx:
        x, y = p % W, p // W
        for q, ok in ((p + 1, x + 1 < W), (p + W, y + 1 < H)):
            if ok and inm[q] and abs(v[q] - v[p]) <= rtol * abs(v[p]):
                amb[p] = amb[q] = True
    return ~amb[idx]


def test_tv_loss(ctx, G, si):
    # the raster is passed as v - v0 (fp32 keeps the full relative precision)
    val, grad = ctx.tv_loss(si.grid, si.mask, _dev(G), si.cfg.lambda_tv)
    assert abs(val - float(G["tv_value"])) <= LOSS_TOL * abs(float(G["tv_value"]))
    keep = tv_unambiguous(si.grid, si.mask, G["sos"])
    assert keep.mean() > 0.95
    # gradients are lambda * (sum of signs): compare the integer sign sums
    np.testing.assert_array_equal(np.round(grad.double().cpu().numpy()[keep] / si.cfg.lambda_tv),
                                  np.round(G["tv_grad"][keep] / si.cfg.lambda_tv))


def test_siren_backward(ctx, G, si):
    cfg = si.cfg
    spec = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, 1500.0)
    g = torch.as_tensor(G["grad_v_masked"].astype(np.float32)).cuda()
    grad = ctx.siren_backward(spec, torch.as_tensor(G["theta2"]), si.grid, si.mask, g)
    err = rel_l2(grad.cpu().numpy(), G["grad_theta"])
    assert err <= GRAD_TOL, err


def test_deconvolve_image(ctx, G, si):
    cfg = si.cfg
    lay = make_patch_layout(si.grid, cfg.patch_mm, cfg.overlap)
    stack = torch.as_tensor(G["stack"].astype(np.float32)).cuda()
    img = ctx.deconvolve_image(stack, cfg.delays, 1500.0, _dev(G), si.ring, si.mask, lay,
                               DeconvolveOptions(cfg.eps_deconv, cfg.n_angles, cfg.ray_step,
                                                 cfg.merge_fwhm))
    err = rel_l2(img.double().cpu().numpy(), G["deconv"])
    assert err <= IMG_TOL, err


def test_one_iteration_loss_and_gradient(ctx, G, si):
    cfg = replace(si.cfg, seed=2, epochs=1, steps_per_epoch=1)
    sig = torch.as_tensor(G["sig"]).cuda()
    tr = Trainer(ctx, sig, si.ring, _meta(G), si.grid, si.mask, cfg)
    tr.step(1)
    data, tv, total = tr.report(1)
    assert abs(data - float(G["data_term"])) <= LOSS_TOL * abs(float(G["data_term"]))
    assert abs(tv - float(G["tv_term"])) <= LOSS_TOL * abs(float(G["tv_term"]))
    g = tr.read(6, (tr.n_params,), np.float64)
    err = rel_l2(g, G["grad_theta"])
    assert err <= GRAD_TOL, err
    tr.close()


def test_joint_reconstruct_matches_reference(ctx, G, si):
    cfg = replace(si.cfg, epochs=3, steps_per_epoch=2, seed=5)
    sig = torch.as_tensor(G["sig"]).cuda()
    reps, img, sos, th = joint_reconstruct(ctx, sig, si.ring, _meta(G), si.grid, si.mask, cfg)
    want = G["reports"]
    assert rel_l2(reps[:, 0], want[:, 0]) <= LOSS_TOL
    assert rel_l2(reps[:, 1], want[:, 1]) <= LOSS_TOL
    assert rel_l2(reps[:, 2], want[:, 2]) <= LOSS_TOL
    assert rel_l2(th, G["joint_theta"]) <= GRAD_TOL
    assert rel_l2(sos.double().cpu().numpy() - 1500.0, G["joint_sos"] - 1500.0) <= 1e-3
    assert rel_l2(img.double().cpu().numpy(), G["joint_image"]) <= IMG_TOL


def test_training_is_deterministic(ctx, G, si):
    # test_optimize.cpp:262-278
    cfg = replace(si.cfg, epochs=3, steps_per_epoch=2, seed=5)
    sig = torch.as_tensor(G["sig"]).cuda()
    a = joint_reconstruct(ctx, sig, si.ring, _meta(G), si.grid, si.mask, cfg)
    b = joint_reconstruct(ctx, sig, si.ring, _meta(G), si.grid, si.mask, cfg)
    assert np.array_equal(a[0][:, :3], b[0][:, :3])
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    assert np.array_equal(a[3], b[3])
    for e in range(3):
        assert a[0][e, 2] == pytest.approx(a[0][e, 0] + a[0][e, 1], rel=1e-12)


def test_batched_joint_reconstruct_equals_separate_calls(ctx, G, si):
    from paper_2409_10876_b200.api import joint_reconstruct_batch

    cfgs = [replace(si.cfg, epochs=2, steps_per_epoch=2, seed=s) for s in (5, 7, 9)]
    sig = torch.as_tensor(G["sig"]).cuda()
    reps, imgs, soss, ths = joint_reconstruct_batch(ctx, [sig, sig, sig], si.ring, _meta(G),
                                                    si.grid, si.mask, cfgs)
    for f, cfg in enumerate(cfgs):
        r, img, sos, th = joint_reconstruct(ctx, sig, si.ring, _meta(G), si.grid, si.mask, cfg)
        assert np.array_equal(reps[f][:, :3], r[:, :3])
        assert torch.equal(imgs[f], img) and torch.equal(soss[f], sos)
        assert np.array_equal(ths[f], th)


def test_batched_joint_reconstruct_with_host_buffers(ctx, G, si):
    """Pinned host signals and outputs (staged by the engine on each frame's
    stream) give the results of the device-buffer call bitwise."""
    from paper_2409_10876_b200.api import joint_reconstruct_batch

    cfgs = [replace(si.cfg, epochs=2, steps_per_epoch=1, seed=s) for s in (5, 7)]
    sig = torch.as_tensor(G["sig"])
    dev = joint_reconstruct_batch(ctx, [sig.cuda(), sig.cuda()], si.ring, _meta(G), si.grid, si.mask,
                                  cfgs)
    hsig = [sig.clone().pin_memory() for _ in cfgs]
    himg = [torch.zeros((si.grid.height, si.grid.width), dtype=torch.float32).pin_memory()
            for _ in cfgs]
    hsos = [torch.zeros_like(t).pin_memory() for t in himg]
    reps, _, _, ths = joint_reconstruct_batch(ctx, hsig, si.ring, _meta(G), si.grid, si.mask, cfgs,
                                              images=himg, sos=hsos)
    torch.cuda.synchronize()
    assert np.array_equal(reps[:, :, :3], dev[0][:, :, :3]) and np.array_equal(ths, dev[3])
    for f in range(len(cfgs)):
        assert torch.equal(himg[f], dev[1][f].cpu()) and torch.equal(hsos[f], dev[2][f].cpu())
    # pageable host signals work too (a synchronous staged copy)
    r2 = joint_reconstruct_batch(ctx, [sig.clone(), sig.clone()], si.ring, _meta(G), si.grid,
                                 si.mask, cfgs)
    assert torch.equal(r2[1][0], dev[1][0]) and np.array_equal(r2[3], dev[3])
