"""GPU metrics of the evaluation harness (evaluate.hpp:39-114)
against the reference's values (tests/golden/metrics.npz via oracle/_ref) and the
reference's own known-answer tests (test_evaluate.cpp:38-112), plus the
benchmark harness (evaluate.hpp:164-220; test_evaluate.cpp:114-139).
"""
import math

import numpy as np
import pytest
import torch

import golden_util as gu
from paper_2409_10876_b200 import evaluate as ev
from paper_2409_10876_b200._abi import ValidationError
from paper_2409_10876_b200.api import (CircularMask, GridSpec, RingGeometry, SignalMetaInfo)

pytestmark = pytest.mark.gpu


def test_matches_reference(ctx):
    z = gu.load("metrics")
    got = [ev.psnr(ctx, z["b"], z["a"], 1.0), ev.ssim(ctx, z["b"], z["a"], 1.0),
           ev.psnr(ctx, z["shifted"], z["img"], 1.0), ev.ssim(ctx, z["shifted"], z["img"], 1.0),
           ev.sos_rmse_masked(ctx, z["sos_r"], z["sos_t"], gu.grid(z["grid"]), gu.mask(z["mask"]))]
    np.testing.assert_allclose(got, z["vals"], rtol=1e-11)


def _random(n, seed):
    return np.random.default_rng(seed).uniform(0, 1, (n, n))


def test_psnr_known_answers(ctx):
    truth = _random(32, 1)
    assert math.isinf(ev.psnr(ctx, truth, truth, 1.0))
    assert abs(ev.psnr(ctx, truth + 0.1, truth, 1.0) - 20.0) <= 1e-9
    binary = np.zeros((32, 32))
    binary[:, :16] = 1.0
    assert abs(ev.psnr(ctx, np.zeros((32, 32)), binary, 1.0) - 10 * math.log10(2.0)) <= 1e-9
    with pytest.raises(ValidationError, match="psnr: image shapes differ"):
        ev.psnr(ctx, truth, _random(16, 2), 1.0)
    with pytest.raises(ValidationError, match="psnr: data_range must be > 0"):
        ev.psnr(ctx, truth, truth, 0.0)


def test_ssim_known_answers(ctx):
    truth = _random(32, 3)
    assert abs(ev.ssim(ctx, truth, truth, 1.0) - 1.0) <= 1e-12
    iy, ix = np.mgrid[0:32, 0:32]
    zm = 0.5 * np.sin(2.1 * ix) * np.cos(1.9 * iy)
    assert ev.ssim(ctx, -zm, zm, 1.0) <= 0.0
    c1, c2, C1 = 0.4, 0.6, 0.01 ** 2
    want = (2 * c1 * c2 + C1) / (c1 * c1 + c2 * c2 + C1)
    assert abs(ev.ssim(ctx, np.full((16, 16), c2), np.full((16, 16), c1), 1.0) - want) <= 1e-9
    with pytest.raises(ValidationError, match="ssim: images must be at least 11x11"):
        ev.ssim(ctx, _random(8, 4), _random(8, 4), 1.0)


def test_shift_is_penalised(ctx):
    z = gu.load("metrics")
    img, shifted = z["img"], z["shifted"]
    assert ev.psnr(ctx, shifted, img, 1.0) < ev.psnr(ctx, img, img, 1.0)
    assert ev.ssim(ctx, shifted, img, 1.0) < ev.ssim(ctx, img, img, 1.0) - 0.05
    assert ev.psnr(ctx, shifted, img, 1.0) < 30.0


def test_masked_sos_rmse(ctx):
    g = GridSpec.centered(33, 33, 0.1)
    val = ev.sos_rmse_masked(ctx, np.full((33, 33), 1510.0), np.full((33, 33), 1500.0), g,
                             CircularMask(0.0, 0.0, 1.0))
    assert abs(val - 10.0) <= 1e-12
    with pytest.raises(ValidationError, match="sos_rmse: mask covers no pixels"):
        ev.sos_rmse_masked(ctx, np.zeros((33, 33)), np.zeros((33, 33)), g,
                           CircularMask(40.0, 40.0, 0.01))


def test_benchmark_single_method(ctx):
    # test_evaluate.cpp:114-139 with the phantom rasterised directly: a 1.5 mm
    # disc at 1540 m/s and two point targets inside a 2.5 mm mask
    grid = GridSpec.centered(65, 65, 0.1)
    ring = RingGeometry(64, 50.0, 0.0)
    xs = grid.origin_x + np.arange(65) * 0.1
    X, Y = np.meshgrid(xs, xs)
    sos = np.where(np.hypot(X - 0.3, Y + 0.2) <= 1.5, 1540.0, 1500.0)
    pressure = np.zeros((65, 65))
    pressure[32, 32] = 1.0
    pressure[37, 42] = 0.7
    truth = ev.Phantom(grid, pressure, sos, CircularMask(0.0, 0.0, 2.5), 1500.0)
    meta = SignalMetaInfo(800, 25e-9, 28e-6, 1500.0)
    sig = ctx.simulate_signals(grid, pressure, sos, truth.mask, 1500.0, ring, meta)
    cfg = ev.BenchmarkConfig(grid=grid, das_v0=1500.0)
    entries = ev.benchmark(ctx, sig, ring, meta, truth, ["das"], cfg)
    assert len(entries) == 1
    r = entries[0].report
    assert r.method == "das" and math.isfinite(r.psnr) and r.ssim <= 1.0 and r.runtime > 0.0
    assert 10.0 < r.psnr < 60.0
    assert 10.0 < r.sos_rmse < 40.0  # implied uniform map vs the disc inclusion
    with pytest.raises(ValidationError, match="benchmark: unknown method 'apact'"):
        ev.benchmark(ctx, sig, ring, meta, truth, ["apact"], cfg)
