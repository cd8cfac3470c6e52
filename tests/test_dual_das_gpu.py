"""GPU parity of dual_sos_das (beamform.hpp:124-150) against the
reference's output (tests/golden/dual_das.npz, generated through oracle/_ref),
plus the reference's own known-answer tests (test_beamform.cpp:133-165):
body_sos = v0 degenerates to plain DAS, and the true body SOS refocuses a
point source that plain DAS smears onto a ring.  Tolerance: 1e-5 relative
L2 (the DAS bar of BASELINE north_star is 1e-4).
"""
import numpy as np
import pytest
import torch

import golden_util as gu
from oracle_lib import rel_l2
from paper_2409_10876_b200._abi import ValidationError
from paper_2409_10876_b200.api import (BodyModel, CircularMask, GridSpec, RingGeometry,
                                       SignalMetaInfo)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Z():
    return gu.load("dual_das")


def test_matches_reference(ctx, Z):
    sig = torch.as_tensor(Z["sig"]).cuda()
    for b, want in zip(Z["bodies"], Z["out"]):
        out = ctx.dual_sos_das(sig, gu.ring(Z["ring"]), gu.meta(Z["meta"]), gu.grid(Z["grid"]),
                               float(Z["v0"]), BodyModel(*map(float, b)))
        err = rel_l2(out.double().cpu().numpy(), want)
        assert err <= 1e-5, err


def test_body_at_v0_is_plain_das(ctx, Z):
    sig = torch.as_tensor(Z["sig"]).cuda()
    ring, meta, grid = gu.ring(Z["ring"]), gu.meta(Z["meta"]), gu.grid(Z["grid"])
    a = ctx.dual_sos_das(sig, ring, meta, grid, 1500.0, BodyModel(0.0, 0.0, 8.0, 1500.0))
    b = ctx.das(sig, ring, meta, grid, 1500.0, 0.0)
    scale = b.abs().max().item()
    assert (a - b).abs().max().item() <= 1e-5 * scale


def test_validation_messages(ctx, Z):
    sig = torch.as_tensor(Z["sig"]).cuda()
    ring, meta, grid = gu.ring(Z["ring"]), gu.meta(Z["meta"]), gu.grid(Z["grid"])
    cases = [(BodyModel(0.0, 0.0, 0.0, 1500.0), 1500.0, "body model: radius must be > 0"),
             (BodyModel(0.0, 0.0, 5.0, 1900.0), 1500.0, "body model: SOS outside [1300, 1800] m/s"),
             (BodyModel(0.0, 0.0, 5.0, 1500.0), 0.0, "dual_sos_das: v0 must be > 0"),
             (BodyModel(20.0, 0.0, 15.0, 1500.0), 1500.0,
              "dual_sos_das: body disc extends outside the transducer ring")]
    for body, v0, msg in cases:
        with pytest.raises(ValidationError, match=msg.replace("[", r"\[").replace("]", r"\]")):
            ctx.dual_sos_das(sig, ring, meta, grid, v0, body)


def test_true_body_sos_refocuses_point_source(ctx):
    # test_beamform.cpp:143-165: a point source at the centre of an 8 mm disc at
    # 1580 m/s, ring of 128 at 50 mm; plain DAS at 1500 m/s puts the peak on a
    # ring, dual-SOS DAS with the true body puts it back on the centre pixel.
    ring = RingGeometry(128, 50.0, 0.0)
    sim_grid = GridSpec.centered(255, 255, 0.1)
    xs = sim_grid.origin_x + np.arange(255) * 0.1
    X, Y = np.meshgrid(xs, xs)
    sos = np.where(np.hypot(X, Y) <= 8.0, 1580.0, 1500.0)
    pressure = np.zeros((255, 255))
    pressure[127, 127] = 1.0
    meta = SignalMetaInfo(1200, 25e-9, 25e-6, 1500.0)
    sig = ctx.simulate_signals(sim_grid, pressure, sos, CircularMask(0.0, 0.0, 49.0), 1500.0,
                               ring, meta)
    grid = GridSpec.centered(65, 65, 0.1)
    plain = ctx.das(sig, ring, meta, grid, 1500.0, 0.0).abs().cpu().numpy()
    fixed = ctx.dual_sos_das(sig, ring, meta, grid, 1500.0,
                             BodyModel(0.0, 0.0, 8.0, 1580.0)).abs().cpu().numpy()
    py, px = np.unravel_index(np.argmax(plain), plain.shape)
    assert (px, py) != (32, 32)
    fy, fx = np.unravel_index(np.argmax(fixed), fixed.shape)
    assert (fx, fy) == (32, 32)
