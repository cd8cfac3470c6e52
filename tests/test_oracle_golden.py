"""CPU: the C restatement (oracle/pact_oracle.c) reproduces the reference's
own outputs (tests/golden, generated through oracle/_ref from the unmodified
reference headers).  This pins the oracle before it is trusted as checker."""
from dataclasses import replace

import numpy as np
import pytest

import golden_util as gu
from oracle_lib import orc, ref, rel_l2
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import SirenSpec

TIGHT = 1e-10  # same fp64 algorithm: agreement to rounding


@pytest.mark.parametrize("name", ["das_edge", "das_cfg1_crop"])
def test_das_stack_restatement_matches_reference(name):
    z = gu.load(name)
    out = orc().das_stack(z["sig"].astype(np.float64), gu.ring(z["ring"]), gu.meta(z["meta"]),
                          gu.grid(z["grid"]), float(z["v0"]), z["delays"])
    assert np.abs(out - z["out"]).max() <= 1e-12 * max(1.0, np.abs(z["out"]).max())


def test_dual_sos_das_restatement_matches_reference():
    from paper_2409_10876_b200.api import BodyModel

    z = gu.load("dual_das")
    for b, want in zip(z["bodies"], z["out"]):
        body = BodyModel(*map(float, b))
        out = orc().dual_sos_das(z["sig"].astype(np.float64), gu.ring(z["ring"]),
                                 gu.meta(z["meta"]), gu.grid(z["grid"]), float(z["v0"]), body)
        assert np.abs(out - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
    # the body disc changes the image (the fixture is not a plain-DAS case)
    plain = orc().das_stack(z["sig"].astype(np.float64), gu.ring(z["ring"]), gu.meta(z["meta"]),
                            gu.grid(z["grid"]), float(z["v0"]), [0.0])[0]
    assert rel_l2(plain, z["out"][0]) > 0.1


def test_metrics_restatement_matches_reference():
    z = gu.load("metrics")
    o = orc()
    got = [o.psnr(z["b"], z["a"], 1.0), o.ssim(z["b"], z["a"], 1.0),
           o.psnr(z["shifted"], z["img"], 1.0), o.ssim(z["shifted"], z["img"], 1.0),
           o.sos_rmse_masked(z["sos_r"], z["sos_t"], gu.grid(z["grid"]), gu.mask(z["mask"]))]
    np.testing.assert_allclose(got, z["vals"], rtol=1e-12)


def test_das_edge_fixture_exercises_both_window_edges():
    z = gu.load("das_edge")
    m = gu.meta(z["meta"])
    g = gu.grid(z["grid"])
    r = gu.ring(z["ring"])
    pos = r.positions()
    xs, ys = g.world(np.arange(g.width), np.arange(g.height))
    X, Y = np.meshgrid(xs, ys)
    dist = np.hypot(X[..., None] - pos[:, 0], Y[..., None] - pos[:, 1])
    s = (1e-3 * (dist[..., None] - z["delays"]) / float(z["v0"]) - m.t0) / m.dt
    assert (s < 0).any() and (s > m.n_samples - 1).any() and ((s >= 0) & (s <= m.n_samples - 1)).any()


@pytest.fixture(scope="module")
def G():
    return gu.load("small_instance")


@pytest.fixture(scope="module")
def si():
    return gu.small_instance()


def _spec(si):
    c = si.cfg
    return SirenSpec(c.hidden, c.sine_layers, c.omega0, c.out_scale, 1500.0)


def test_init_siren_bitwise(G, si):
    s = _spec(si)
    assert np.array_equal(orc().init_siren(0, s, s.param_count()), G["theta0"])
    assert np.array_equal(orc().init_siren(2, s, s.param_count()), G["theta2"])


def test_init_siren_matches_library_and_reference_counts(si):
    # test_nfield.cpp:26-46 parameter counts
    from paper_2409_10876_b200.api import init_siren

    assert SirenSpec(64, 2).param_count() == 4417
    assert SirenSpec(16, 2).param_count() == 337
    s = _spec(si)
    assert np.array_equal(init_siren(2, s), orc().init_siren(2, s, s.param_count()))


def test_render_and_backprop(G, si):
    s = _spec(si)
    sos = orc().render_sos(s, G["theta2"], si.grid, si.mask)
    assert rel_l2(sos, G["sos"]) <= TIGHT
    g = orc().backprop_sos(s, G["theta2"], si.grid, si.mask, G["grad_v_masked"])
    assert rel_l2(g, G["grad_theta"]) <= 1e-9


def test_wavefront_transfer_spectra(G, si):
    c = si.cfg
    lay = orc().patch_layout(si.grid, c.patch_mm, c.overlap)
    w = orc().wavefront_profile(lay["centers"], si.ring, si.grid, G["sos"], 1500.0, si.mask,
                                c.n_angles, c.ray_step)
    assert rel_l2(w, G["w"]) <= TIGHT
    H = orc().transfer_stack(G["w"][0], c.delays, lay["P"], si.grid.pitch)
    assert rel_l2(H, G["H0"]) <= TIGHT
    Y = orc().patch_spectra(G["stack"], c.delays, 1500.0, si.grid, c.patch_mm, c.overlap)
    assert rel_l2(Y, G["Y"]) <= 1e-7  # fixture stores Y as complex64


def test_fused_loss_trace_tv(G, si):
    c = si.cfg
    lay = orc().patch_layout(si.grid, c.patch_mm, c.overlap)
    n, K = G["Y"].shape[:2]
    P = lay["P"]
    scale = 1.0 / (n * K * P * P)
    gv = np.zeros((si.grid.height, si.grid.width))
    for i in range(n):
        loss, dw = orc().fused_patch_loss_grad(G["Y"][i], G["w"][i], P, si.grid.pitch, c.n_angles,
                                               c.delays, c.eps_deconv, scale)
        assert abs(loss - G["loss_patch"][i]) <= 1e-9 * abs(G["loss_patch"][i])
        assert rel_l2(dw, G["dw"][i]) <= 1e-9
        gv = orc().wavefront_grad_trace(lay["centers"][i], si.ring, si.grid, G["sos"], 1500.0,
                                        si.mask, c.n_angles, c.ray_step, G["dw"][i], gv)
    val, tvg = orc().tv_loss(si.grid, G["sos"], si.mask, c.lambda_tv)
    assert val == pytest.approx(float(G["tv_value"]), rel=1e-12)
    assert rel_l2(tvg, G["tv_grad"]) <= TIGHT
    from paper_2409_10876_b200.api import masked_pixels

    idx, _ = masked_pixels(si.grid, si.mask)
    assert rel_l2(gv.ravel()[idx] + tvg, G["grad_v_masked"]) <= 1e-9


def test_nf_step_and_deconvolution(G, si):
    meta = gu.meta(G["meta"])
    sig = G["sig"].astype(np.float64)
    out = orc().nf_step(sig, si.ring, meta, si.grid, si.mask, replace(si.cfg, seed=2),
                        G["theta2"])
    assert out["data_term"] == pytest.approx(float(G["data_term"]), rel=1e-9)
    assert out["tv_term"] == pytest.approx(float(G["tv_term"]), rel=1e-12)
    assert rel_l2(out["grad_theta"], G["grad_theta"]) <= 1e-8
    assert rel_l2(out["image"], G["image"]) <= 1e-9
    c = si.cfg
    img = orc().deconvolve_image(G["stack"], c.delays, 1500.0, si.grid, G["sos"], si.ring,
                                 si.mask, c.patch_mm, c.overlap, c.eps_deconv, c.n_angles,
                                 c.ray_step, c.merge_fwhm)
    assert rel_l2(img, G["deconv"]) <= 1e-9


def test_joint_reconstruct(G, si):
    meta = gu.meta(G["meta"])
    cfg = replace(si.cfg, epochs=3, steps_per_epoch=2, seed=5)
    reps, img, sos, th = orc().joint_reconstruct(G["sig"].astype(np.float64), si.ring, meta,
                                                 si.grid, si.mask, cfg, _spec(si).param_count())
    assert rel_l2(reps[:, :3], G["reports"][:, :3]) <= 1e-8
    assert rel_l2(th, G["joint_theta"]) <= 1e-8
    assert rel_l2(img, G["joint_image"]) <= 1e-8
    assert rel_l2(sos, G["joint_sos"]) <= 1e-12


def test_adam_known_answers():
    # test_optimize.cpp:27-66
    p, m, v, t = orc().adam_step([1.0, -2.0, 0.5], [0.0, 0.0, 0.0], [0] * 3, [0] * 3, 0, 1e-3,
                                 0.9, 0.999, 1e-8)
    assert t == 1 and list(p) == [1.0, -2.0, 0.5]
    p, m, v, t = orc().adam_step([0.0, 0.0], [3.7, -0.002], [0, 0], [0, 0], 0, 1e-3, 0.9, 0.999,
                                 1e-8)
    assert p[0] == pytest.approx(-1e-3, rel=1e-4) and p[1] == pytest.approx(1e-3, rel=1e-2)
    with pytest.raises(RuntimeError):
        orc().adam_step([0.0], [float("nan")], [0], [0], 0, 1e-3, 0.9, 0.999, 1e-8)


def test_cfg2_step_restatement():
    """cfg2 (BASELINE configs[1]) forward + gradient from the fixture signals."""
    z = gu.load("cfg2_step")
    w = wl.cfg2()
    cfg = wl.train_config(w)
    out = orc().nf_step(z["sig"].astype(np.float64), w.ring, w.meta, w.grid, w.mask, cfg,
                        z["theta"], want_image=False)
    assert out["data_term"] == pytest.approx(float(z["data_term"]), rel=1e-9)
    assert out["tv_term"] == pytest.approx(float(z["tv_term"]), rel=1e-9)
    assert rel_l2(out["w"], z["w"]) <= 1e-10
    assert rel_l2(out["grad_theta"], z["grad_theta"]) <= 1e-8


def test_reference_shim_available_here_or_skipped():
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built (no /root/reference on this machine)")
    z = gu.load("das_edge")
    out = R.das_stack(z["sig"], gu.ring(z["ring"]), gu.meta(z["meta"]), gu.grid(z["grid"]),
                      float(z["v0"]), z["delays"], workers=1)
    assert rel_l2(out, z["out"]) == 0.0
