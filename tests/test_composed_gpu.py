"""GPU parity of the composed (non-fused) path (csrc/composed.cu, fp64)
against the reference itself (oracle/_ref), plus the reference's own
finite-difference contracts for it, run through the GPU entry points:

  multichannel_deconvolve   deconv.hpp:78-96
  deconv_jacobian_H         deconv.hpp:100-115   (FD: test_deconv.cpp:149-181)
  patch_data_loss/data_loss optimize.hpp:155-211, 329-353  (FD: test_optimize.cpp:157-203)
  transfer_grad_to_wavefront aberration.hpp:270-313
  wavefront_profile(with_jacobian) + accumulate_wavefront_grad  aberration.hpp:134-186, 316-326
  merge_patches             deconv.hpp:118-164
  psf_from_transfer         aberration.hpp:407-445
  full_chain_grad == the fused training gradient (test_support.hpp:95-118;
  test_optimize.cpp:306-351), on the reference's SmallInstance
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import golden_util as gu
from oracle_lib import ref, rel_l2
from paper_2409_10876_b200.api import (SirenSpec, make_delays, make_patch_layout)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    r = ref()
    if r is None:
        pytest.skip("oracle/_ref/libpact_ref.so not built")
    return r


def _rand_spectra(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _cu(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.complex128)).cuda()


@pytest.mark.parametrize("P", [8, 7])
def test_multichannel_deconvolve(ctx, R, P):
    rng = np.random.default_rng(3)
    n, K = 3, 4
    Y, H = _rand_spectra(rng, (n, K, P, P)), _rand_spectra(rng, (n, K, P, P))
    X = ctx.multichannel_deconvolve(_cu(Y), _cu(H), 1e-3).cpu().numpy()
    for i in range(n):
        assert rel_l2(X[i], R.multichannel_deconvolve(Y[i], H[i], 1e-3)) <= 1e-13


def test_deconv_jacobian_matches_reference_and_fd(ctx, R):
    """deconv_jacobian_H vs the reference, and vs central differences of the
    GPU multichannel_deconvolve (test_deconv.cpp:149-181: h = 1e-6, 1e-4)."""
    rng = np.random.default_rng(9)
    K, P = 3, 8
    Y, H = _rand_spectra(rng, (1, K, P, P)), _rand_spectra(rng, (1, K, P, P))
    q = [(0, int(rng.integers(K)), int(rng.integers(P * P))) for _ in range(20)]
    J = ctx.deconv_jacobian_H(_cu(Y), _cu(H), 1e-3, q).cpu().numpy()
    h = 1e-6
    for t, (_, j, b) in enumerate(q):
        dre, dim = R.deconv_jacobian_H(Y[0], H[0], 1e-3, j, b)
        assert abs(J[t, 0] - dre) <= 1e-12 * max(1.0, abs(dre))
        assert abs(J[t, 1] - dim) <= 1e-12 * max(1.0, abs(dim))
        fd = []
        for d in (h, 1j * h):
            hp, hm = H.copy(), H.copy()
            hp[0, j].flat[b] += d
            hm[0, j].flat[b] -= d
            xp = ctx.multichannel_deconvolve(_cu(Y), _cu(hp), 1e-3).cpu().numpy()[0].flat[b]
            xm = ctx.multichannel_deconvolve(_cu(Y), _cu(hm), 1e-3).cpu().numpy()[0].flat[b]
            fd.append((xp - xm) / (2 * h))
        scale = max(1.0, abs(J[t, 0]) + abs(J[t, 1]))
        assert abs(fd[0] - J[t, 0]) < 1e-4 * scale
        assert abs(fd[1] - J[t, 1]) < 1e-4 * scale


@pytest.mark.parametrize("P,implicit", [(8, True), (8, False), (7, True)])
def test_patch_and_data_loss_vs_reference(ctx, R, P, implicit):
    rng = np.random.default_rng(11)
    n, K, pitch = 2, 3, 0.1
    Y, H = _rand_spectra(rng, (n, K, P, P)), _rand_spectra(rng, (n, K, P, P))
    scale = 0.37
    loss, g = ctx.patch_data_loss(_cu(Y), _cu(H), pitch, 1e-3, scale, implicit)
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    for i in range(n):
        lv, gr = R.patch_data_loss(Y[i], H[i], pitch, 1e-3, scale, implicit)
        assert abs(loss[i] - lv) <= 1e-12 * abs(lv)
        assert rel_l2(g[i], gr) <= 1e-12
    val, per, gd = ctx.data_loss(_cu(Y), _cu(H), pitch, 1e-3, implicit)
    rv, rg = R.data_loss(Y, H, pitch, 1e-3, implicit)
    assert abs(val - rv) <= 1e-12 * abs(rv)
    assert abs(per.sum().item() - rv) <= 1e-12 * abs(rv)
    assert rel_l2(gd.cpu().numpy(), rg) <= 1e-12


def test_data_loss_grad_h_finite_differences(ctx):
    """test_optimize.cpp:157-203 through the GPU: transfer_stack of a random
    profile, random real-patch spectra, dL/dH vs central differences (h = 1e-6,
    1e-4 of max(1, |fd|)).  The profile's H comes from the reference formula
    in fp64 here (the GPU transfer_stack is fp32; this checks the loss)."""
    rng = np.random.default_rng(19)
    P, M, pitch, A = 8, 3, 0.1, 16
    w = 0.2 * rng.uniform(-1, 1, A)
    d = make_delays(-0.25, 0.25, M)
    H = np.zeros((1, M, P, P), np.complex128)
    sc = 2 * np.pi / (P * pitch)
    for by in range(P):
        for bx in range(P):
            kx = sc * (bx if bx <= P // 2 else bx - P)
            ky = sc * (by if by <= P // 2 else by - P)
            k, ang = np.hypot(kx, ky), np.arctan2(ky, kx)
            if k == 0:
                H[0, :, by, bx] = 1
                continue

            def wi(t):
                pos = np.fmod(t, 2 * np.pi)
                pos = pos + 2 * np.pi if pos < 0 else pos
                pos = pos / (2 * np.pi) * A
                a0 = int(pos) % A
                f = pos - np.floor(pos)
                return (1 - f) * w[a0] + f * w[(a0 + 1) % A]
            w1, w2 = wi(ang), wi(ang + np.pi)
            for j in range(M):
                H[0, j, by, bx] = 0.5 * np.exp(-1j * k * (d[j] - w1)) + 0.5 * np.exp(1j * k * (d[j] - w2))
    Y = np.fft.fft2(rng.uniform(-1, 1, (1, M, P, P)))
    _, _, g = ctx.data_loss(_cu(Y), _cu(H), pitch, 1e-3, True)
    g = g.cpu().numpy()
    h = 1e-6
    for _ in range(12):
        b = int(rng.integers(P * P))
        j = int(rng.integers(M))

        def val(delta):
            hp = H.copy()
            hp[0, j].flat[b] += delta
            return ctx.data_loss(_cu(Y), _cu(hp), pitch, 1e-3, True)[0]
        fd_re = (val(h) - val(-h)) / (2 * h)
        fd_im = (val(1j * h) - val(-1j * h)) / (2 * h)
        gb = g[0, j].flat[b]
        scale = max(1.0, abs(fd_re), abs(fd_im))
        assert abs(gb.real - fd_re) <= 1e-4 * scale
        assert abs(gb.imag - fd_im) <= 1e-4 * scale


@pytest.mark.parametrize("P,A", [(8, 16), (64, 512), (7, 32)])
def test_transfer_grad_to_wavefront_vs_reference(ctx, R, P, A):
    rng = np.random.default_rng(P + A)
    n, K, pitch = 2, 4, 0.1
    d = make_delays(-1.0, 1.0, K)
    w = 0.3 * rng.uniform(-1, 1, (n, A))
    g = _rand_spectra(rng, (n, K, P, P))
    dw = ctx.transfer_grad_to_wavefront(torch.as_tensor(w).cuda(), d, P, pitch, _cu(g)).cpu().numpy()
    for i in range(n):
        want = R.transfer_grad_to_wavefront(w[i], d, P, pitch, g[i])
        assert rel_l2(dw[i], want) <= 1e-11


@pytest.fixture(scope="module")
def G():
    return gu.load("small_instance")


@pytest.fixture(scope="module")
def si():
    return gu.small_instance()


def test_wavefront_jacobian_and_accumulate(ctx, R, G, si):
    """Sparse Jacobian rows of every SmallInstance patch vs the reference's
    (same row lengths, same pixels in the same order, dw/dv to fp32), the
    profiles, and J^T dw."""
    lay = make_patch_layout(si.grid, si.cfg.patch_mm, si.cfg.overlap)
    sos = G["sos"].astype(np.float32).astype(np.float64)  # fp32-representable for both sides
    dev = torch.as_tensor((sos - 1500.0).astype(np.float32)).cuda()
    A, step = si.cfg.n_angles, si.cfg.ray_step
    w, rs, pix, val = ctx.wavefront_jacobian(si.ring, si.grid, dev, 1500.0, si.mask, lay.centers,
                                             A, step)
    w, rs, pix, val = (t.cpu().numpy() for t in (w, rs, pix, val))
    rng = np.random.default_rng(5)
    dw = rng.standard_normal((lay.n_patches, A))
    gv = torch.zeros((si.grid.height, si.grid.width), device="cuda", dtype=torch.float64)
    ctx.accumulate_wavefront_grad(torch.as_tensor(rs).cuda(), torch.as_tensor(pix).cuda(),
                                  torch.as_tensor(val).cuda(), torch.as_tensor(dw.ravel()).cuda(), gv)
    gv_ref = np.zeros((si.grid.height, si.grid.width))
    for i in range(lay.n_patches):
        rw, counts, rp, rv, gv_ref = R.wavefront_jacobian(lay.centers[i], si.ring, si.grid, sos,
                                                           1500.0, si.mask, A, step, dw[i], gv_ref)
        assert rel_l2(w[i], rw) <= 1e-6
        lens = np.diff(rs[i * A:(i + 1) * A + 1])
        assert np.array_equal(lens, counts)
        lo, hi = rs[i * A], rs[(i + 1) * A]
        assert np.array_equal(pix[lo:hi], rp)
        assert rel_l2(val[lo:hi], rv) <= 1e-6
    assert rel_l2(gv.cpu().numpy(), gv_ref) <= 1e-6


def test_merge_patches_vs_reference(ctx, R, si):
    lay = make_patch_layout(si.grid, si.cfg.patch_mm, 0.5)
    P = lay.patch_pixels
    rng = np.random.default_rng(2)
    ps = rng.standard_normal((lay.n_patches, P, P)).astype(np.float32)
    img = ctx.merge_patches(lay, torch.as_tensor(ps).cuda(), 1.5).double().cpu().numpy()
    want = R.merge_patches(si.grid, si.cfg.patch_mm, 0.5, ps.astype(np.float64), 1.5)
    assert rel_l2(img, want) <= 1e-6
    ones = ctx.merge_patches(lay, torch.ones((lay.n_patches, P, P), device="cuda"), 1.5)
    assert float((ones - 1).abs().max()) <= 2e-6  # partition of unity (test_deconv.cpp:259-277)


def test_full_chain_grad_equals_fused(ctx, G, si):
    """testsupport::full_chain_grad (test_support.hpp:95-118) composed from the
    GPU entry points — render_sos, wavefront_profile(with_jacobian),
    transfer_stack, patch_data_loss, transfer_grad_to_wavefront,
    accumulate_wavefront_grad, tv_loss, backprop_sos — equals the fused
    training gradient (the reference's nf_step, golden) as in
    test_optimize.cpp:306-351 (there 1e-8 in fp64; here 1e-3, the fp32
    SIREN / ray / H stages)."""
    cfg = si.cfg
    spec = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, 1500.0)
    theta = torch.as_tensor(G["theta2"])  # the golden step's parameters (init_siren seed 2)
    _, dev = ctx.render_sos(spec, theta, si.grid, si.mask)
    lay = make_patch_layout(si.grid, cfg.patch_mm, cfg.overlap)
    P, n, K = lay.patch_pixels, lay.n_patches, len(cfg.delays)
    scale = 1.0 / (n * K * P * P)
    w, rs, pix, val = ctx.wavefront_jacobian(si.ring, si.grid, dev, 1500.0, si.mask, lay.centers,
                                             cfg.n_angles, cfg.ray_step)
    H = ctx.transfer_stack(w.float(), cfg.delays, P, si.grid.pitch).to(torch.complex128)
    Y = torch.as_tensor(G["Y"]).cuda().to(torch.complex128)
    loss, gh = ctx.patch_data_loss(Y, H, si.grid.pitch, cfg.eps_deconv, scale, True)
    assert abs(loss.sum().item() - float(G["data_term"])) <= 1e-3 * abs(float(G["data_term"]))
    dw = ctx.transfer_grad_to_wavefront(w, cfg.delays, P, si.grid.pitch, gh)
    assert rel_l2(dw.cpu().numpy(), G["dw"]) <= 1e-3
    gv = torch.zeros((si.grid.height, si.grid.width), device="cuda", dtype=torch.float64)
    ctx.accumulate_wavefront_grad(rs, pix, val, dw.reshape(-1), gv)
    _, tv_grad = ctx.tv_loss(si.grid, si.mask, dev, cfg.lambda_tv)
    from paper_2409_10876_b200.api import masked_pixels

    idx, _ = masked_pixels(si.grid, si.mask)
    gm = gv.reshape(-1)[torch.as_tensor(idx, dtype=torch.long).cuda()] + tv_grad.double()
    assert rel_l2(gm.cpu().numpy(), G["grad_v_masked"]) <= 1e-3
    grad = ctx.siren_backward(spec, theta, si.grid, si.mask, gm).cpu().numpy()
    err = rel_l2(grad, G["grad_theta"])
    print("composed vs fused grad_theta rel L2", err)
    assert err <= 1e-3


def test_psf_from_transfer_vs_reference(ctx, G, si):
    """Spatial PSFs of the SmallInstance patch-0 transfer stack (reference H,
    golden) vs the reference's psf_from_transfer; the asymmetric-spectrum
    ValidationError carries the reference's text."""
    from cli_helpers import RefIO

    refio = RefIO()
    H = np.ascontiguousarray(G["H0"])  # [K, P, P] complex128, reference transfer_stack
    K, P, _ = H.shape
    psf = ctx.psf_from_transfer(_cu(H)).cpu().numpy()
    for j in range(K):
        rc, want = refio.psf_from_transfer(H[j], P, si.grid.pitch)
        assert rc == 0
        assert np.abs(psf[j] - want).max() <= 1e-12 * np.abs(want).max()
    bad = H[:1].copy()
    bad[0, 1, 2] += 1e-3j
    rc, msg = refio.psf_from_transfer(bad[0], P, si.grid.pitch)
    from paper_2409_10876_b200._abi import ValidationError

    with pytest.raises(ValidationError) as e:
        ctx.psf_from_transfer(_cu(bad))
    assert rc == 2 and str(e.value).endswith(msg)
