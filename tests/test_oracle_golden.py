"""CPU: the C restatement (oracle/pact_oracle.c) reproduces the reference's
own outputs (tests/golden, generated through oracle/_ref from the unmodified
reference headers).  This pins the oracle before it is trusted as checker."""
import numpy as np
import pytest

import golden_util as gu
from oracle_lib import orc, ref, rel_l2


@pytest.mark.parametrize("name", ["das_edge", "das_cfg1_crop"])
def test_das_stack_restatement_matches_reference(name):
    z = gu.load(name)
    out = orc().das_stack(z["sig"].astype(np.float64), gu.ring(z["ring"]), gu.meta(z["meta"]),
                          gu.grid(z["grid"]), float(z["v0"]), z["delays"])
    # same fp64 algorithm: agreement to rounding
    assert np.abs(out - z["out"]).max() <= 1e-12 * max(1.0, np.abs(z["out"]).max())


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


def test_reference_shim_available_here_or_skipped():
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built (no /root/reference on this machine)")
    z = gu.load("das_edge")
    out = R.das_stack(z["sig"], gu.ring(z["ring"]), gu.meta(z["meta"]), gu.grid(z["grid"]),
                      float(z["v0"]), z["delays"], workers=1)
    assert rel_l2(out, z["out"]) == 0.0
