"""§8(f)-3 on the B200: `pactrec` end to end against the reference compiled in
oracle/_ref, on one small scene (twobody phantom, 64 x 64 at 0.3 mm, 96
transducers on a 25 mm ring).

phantom -> simulate (auto window, 1/sqrt(r) spreading) -> recon das / dual-sos /
stack / deconv / nf -> psf dump -> eval.  Each output file is read back and
compared with the reference run on the same inputs (the file values: f32):
  simulate   window bit-exact, samples rel. L2 <= 1e-4 (fp32 device TOF)
  das family rel. L2 <= 1e-5
  deconv     rel. L2 <= 1e-3 (fp32 PSF / FFT path, the §8 image tolerance)
  psf dump   rel. L2 <= 1e-4 per PSF
  nf         files, loss log, SIRN checkpoint loadable by the reference; epoch
             losses within 1e-3 of the reference's joint_reconstruct
"""
import json
import os

import numpy as np
import pytest

import cli_helpers as H
import oracle_lib as O
from paper_2409_10876_b200.api import (BodyModel, CircularMask, GridSpec, RingGeometry,
                                       SignalMetaInfo, TrainConfig)

pytestmark = pytest.mark.gpu
REF = H.ref_io()
ORC_REF = O.ref()
needs_ref = pytest.mark.skipif(REF is None or ORC_REF is None, reason="oracle/_ref not built")

W, PITCH, NTX, RING = 64, 0.3, 96, 25.0
COMMON = ["--grid-size", str(W), "--pitch", str(PITCH)]
SMALL_TRAIN = ["--delays", "-0.5:0.5:4", "--n-angles", "64", "--patch-mm", "4.8", "--overlap", "0.5",
               "--ray-step", "0.1"]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def scene(tmp_path_factory):
    H.build()
    d = tmp_path_factory.mktemp("cli")
    rc, _, se = H.run(["phantom", "--spec", "twobody", *COMMON, "--out", str(d / "ph")], d)
    assert rc == 0, se
    rc, so, se = H.run(["simulate", "--transducers", str(NTX), "--ring-radius", str(RING),
                        "--pressure", str(d / "ph" / "pressure.pgrid"),
                        "--sos", str(d / "ph" / "sos.pgrid"), "--out", str(d / "sim")], d)
    assert rc == 0, se
    return d


def _sig(scene):
    data, (dt, t0, radius, off, bg) = H.read_sigset(str(scene / "sim" / "signals.sigset"))
    ring = RingGeometry(data.shape[0], radius, off)
    meta = SignalMetaInfo(data.shape[1], dt, t0, bg)
    return data.astype(np.float64), ring, meta


@needs_ref
def test_simulate_matches_reference(scene):
    pr, geo = H.read_pgrid(str(scene / "ph" / "pressure.pgrid"))
    so, _ = H.read_pgrid(str(scene / "ph" / "sos.pgrid"))
    bg = REF.water_sos(26.0)
    t0, T, ref = REF.simulate(pr, so, geo, (0.0, 0.0, 10.0), bg, (NTX, RING, 0.0), 100e-9, 25e-9,
                              True, 0.05)
    data, (dt, t0_ours, radius, off, bg_ours) = H.read_sigset(str(scene / "sim" / "signals.sigset"))
    assert data.shape == (NTX, T) and t0_ours == t0 and dt == 25e-9 and bg_ours == bg
    assert rel(data, ref) <= 1e-4, rel(data, ref)


@needs_ref
def test_recon_das_family_matches_reference(scene):
    sig, ring, meta = _sig(scene)
    grid = GridSpec.centered(W, W, PITCH)
    d = scene
    rc, _, se = H.run(["recon", "das", *COMMON, "--signals", str(d / "sim" / "signals.sigset"),
                       "--delay", "0.3", "--out", str(d / "das")], d)
    assert rc == 0, se
    img, geo = H.read_pgrid(str(d / "das" / "image.pgrid"))
    ref = ORC_REF.das_stack(sig, ring, meta, grid, meta.background_sos, [0.3])[0]
    assert geo == (PITCH, grid.origin_x, grid.origin_y)
    assert rel(img, ref) <= 1e-5, rel(img, ref)

    rc, _, se = H.run(["recon", "dual-sos", *COMMON, "--signals", str(d / "sim" / "signals.sigset"),
                       "--body-radius", "8.5", "--body-sos", "1555", "--out", str(d / "dual")], d)
    assert rc == 0, se
    img, _ = H.read_pgrid(str(d / "dual" / "image.pgrid"))
    ref = ORC_REF.dual_sos_das(sig, ring, meta, grid, meta.background_sos,
                               BodyModel(0.0, 0.0, 8.5, 1555.0))
    assert rel(img, ref) <= 1e-5, rel(img, ref)

    rc, so, se = H.run(["recon", "stack", *COMMON, "--signals", str(d / "sim" / "signals.sigset"),
                        "--v0", "1510", "--delays", "-1:1:5", "--out", str(d / "stack")], d)
    assert rc == 0, se
    assert "wrote 5 stack PGRIDs" in so
    ref = ORC_REF.das_stack(sig, ring, meta, grid, 1510.0, np.linspace(-1, 1, 5))
    for j in range(5):
        img, _ = H.read_pgrid(str(d / "stack" / f"stack_{j:03d}.pgrid"))
        assert rel(img, ref[j]) <= 1e-5, (j, rel(img, ref[j]))


@needs_ref
def test_recon_deconv_matches_reference(scene):
    sig, ring, meta = _sig(scene)
    grid = GridSpec.centered(W, W, PITCH)
    d = scene
    rc, _, se = H.run(["recon", "deconv", *COMMON, *SMALL_TRAIN,
                       "--signals", str(d / "sim" / "signals.sigset"),
                       "--sos", str(d / "ph" / "sos.pgrid"), "--out", str(d / "deconv")], d)
    assert rc == 0, se
    img, _ = H.read_pgrid(str(d / "deconv" / "image.pgrid"))
    sos, _ = H.read_pgrid(str(d / "ph" / "sos.pgrid"))
    delays = np.linspace(-0.5, 0.5, 4)
    stack = ORC_REF.das_stack(sig, ring, meta, grid, meta.background_sos, delays)
    ref = ORC_REF.deconvolve_image(stack, delays, meta.background_sos, grid, sos.astype(np.float64),
                                   ring, CircularMask(0.0, 0.0, 10.0), 4.8, 0.5, 1e-3, 64, 0.1, 1.5)
    assert rel(img, ref) <= 1e-3, rel(img, ref)
    # the SOS raster must sit on the reconstruction grid
    rc, _, se = H.run(["recon", "deconv", "--grid-size", "32", "--pitch", str(PITCH),
                       "--signals", str(d / "sim" / "signals.sigset"),
                       "--sos", str(d / "ph" / "sos.pgrid"), "--out", str(d / "deconv2")], d)
    assert rc == 2 and "SOS raster grid does not match" in se


@needs_ref
def test_psf_dump_matches_reference(scene):
    d = scene
    rc, so, se = H.run(["psf", "dump", "--transducers", str(NTX), "--ring-radius", str(RING),
                        *SMALL_TRAIN, "--sos", str(d / "ph" / "sos.pgrid"), "--index", "0", "7",
                        "--out", str(d / "psf")], d)
    assert rc == 0, se
    assert "wrote 8 PSF PGRIDs" in so
    sos, _ = H.read_pgrid(str(d / "ph" / "sos.pgrid"))
    grid = GridSpec.centered(W, W, PITCH)
    lay = ORC_REF.patch_layout(grid, 4.8, 0.5)
    ring = RingGeometry(NTX, RING, 0.0)
    v0 = REF.water_sos(26.0)
    delays = np.linspace(-0.5, 0.5, 4)
    for i in (0, 7):
        w = ORC_REF.wavefront_profile(lay["centers"][i], ring, grid, sos.astype(np.float64), v0,
                                      CircularMask(0.0, 0.0, 10.0), 64, 0.1)[0]
        Hs = ORC_REF.transfer_stack(w, delays, lay["P"], PITCH)
        for j in range(4):
            rc, ref = REF.psf_from_transfer(Hs[j], lay["P"], PITCH)
            assert rc == 0, ref
            psf, geo = H.read_pgrid(str(d / "psf" / f"psf_p{i:04d}_d{j:03d}.pgrid"))
            assert geo == (PITCH, -(lay["P"] // 2) * PITCH, -(lay["P"] // 2) * PITCH)
            assert rel(psf, ref) <= 1e-4, (i, j, rel(psf, ref))
    rc, _, se = H.run(["psf", "dump", "--sos", str(d / "ph" / "sos.pgrid"), "--index", "9999",
                       "--out", str(d / "psf2")], d)
    assert rc == 2 and "patch index out of range: 9999" in se


@needs_ref
def test_recon_nf_outputs_and_losses(scene):
    sig, ring, meta = _sig(scene)
    grid = GridSpec.centered(W, W, PITCH)
    d = scene
    args = ["--epochs", "2", "--steps-per-epoch", "2", "--hidden", "16", "--sine-layers", "2",
            "--seed", "5", "--lambda-tv", "1e8"]
    rc, so, se = H.run(["recon", "nf", *COMMON, *SMALL_TRAIN, *args,
                        "--signals", str(d / "sim" / "signals.sigset"), "--out", str(d / "nf")], d)
    assert rc == 0, se
    for f in ("image.pgrid", "sos.pgrid", "checkpoint.sirn", "loss_log.jsonl", "resolved_config.ini"):
        assert (d / "nf" / f).exists(), f
    log = [json.loads(line) for line in open(d / "nf" / "loss_log.jsonl")]
    assert [r["epoch"] for r in log] == [1, 2]
    assert all(set(r) == {"epoch", "data_term", "tv_term", "total", "seconds"} for r in log)
    rc, (shape, scal, theta) = REF.load_sirn(str(d / "nf" / "checkpoint.sirn"))
    assert rc == 0 and shape == (2, 16, 2) and scal[0] == 30.0
    cfg = TrainConfig(epochs=2, steps_per_epoch=2, hidden=16, sine_layers=2, seed=5,
                      lambda_tv=1e8, delays=list(np.linspace(-0.5, 0.5, 4)), n_angles=64,
                      patch_mm=4.8, overlap=0.5, ray_step=0.1)
    reports, img_ref, sos_ref, _ = ORC_REF.joint_reconstruct(sig, ring, meta, grid,
                                                             CircularMask(0.0, 0.0, 10.0), cfg,
                                                             theta.size)
    for r, rr in zip(log, reports):
        assert abs(r["total"] - rr[2]) <= 1e-3 * abs(rr[2]), (r, rr)
        assert abs(r["data_term"] - rr[0]) <= 1e-3 * abs(rr[0]), (r, rr)
    img, _ = H.read_pgrid(str(d / "nf" / "image.pgrid"))
    assert rel(img, img_ref) <= 1e-3, rel(img, img_ref)


@needs_ref
def test_eval_report(scene):
    d = scene
    rc, so, se = H.run(["eval", *COMMON, "--signals", str(d / "sim" / "signals.sigset"),
                        "--pressure", str(d / "ph" / "pressure.pgrid"),
                        "--sos", str(d / "ph" / "sos.pgrid"), "--methods", "das,dual_sos",
                        "--save-images", "--out", str(d / "eval")], d)
    assert rc == 0, se
    rows = open(d / "eval" / "report.txt").read().splitlines()
    assert rows[0].split() == ["method", "psnr_db", "ssim", "sos_rmse_mps", "runtime_s"]
    vals = {r.split()[0]: [float(x) for x in r.split()[1:]] for r in rows[1:]}
    assert set(vals) == {"das", "dual_sos"}
    for m, (psnr, ssim, rmse, rt) in vals.items():
        assert np.isfinite(psnr) and 0.0 <= ssim <= 1.0 and rmse >= 0 and rt >= 0, (m, vals[m])
    for f in ("das_image.pgrid", "das_sos.pgrid", "dual_sos_image.pgrid", "dual_sos_sos.pgrid"):
        assert (d / "eval" / f).exists()
    # the das image is the conventional DAS at --das-v0 (1510 m/s)
    sig, ring, meta = _sig(scene)
    img, _ = H.read_pgrid(str(d / "eval" / "das_image.pgrid"))
    ref = ORC_REF.das_stack(sig, ring, meta, GridSpec.centered(W, W, PITCH), 1510.0, [0.0])[0]
    assert rel(img, ref) <= 1e-5
    rc, _, se = H.run(["eval", *COMMON, "--signals", str(d / "sim" / "signals.sigset"),
                       "--pressure", str(d / "ph" / "pressure.pgrid"),
                       "--sos", str(d / "ph" / "sos.pgrid"), "--methods", "das,magic",
                       "--out", str(d / "eval2")], d)
    assert rc == 2 and "benchmark: unknown method 'magic'" in se
