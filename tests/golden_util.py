"""Helpers to rebuild API objects from golden fixtures, and the reference's
shared SmallInstance fixture (proj/tests/test_support.hpp:38-75)."""
import os
from dataclasses import dataclass

import numpy as np

from paper_2409_10876_b200.api import (CircularMask, GridSpec, RingGeometry, SignalMetaInfo,
                                       TrainConfig, make_delays)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(name):
    return np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))


def ring(a):
    return RingGeometry(int(a[0]), float(a[1]), float(a[2]))


def grid(a):
    return GridSpec(int(a[0]), int(a[1]), float(a[2]), float(a[3]), float(a[4]))


def meta(a):
    return SignalMetaInfo(int(a[0]), float(a[1]), float(a[2]), float(a[3]))


def mask(a):
    return CircularMask(float(a[0]), float(a[1]), float(a[2]))


@dataclass
class SmallInstance:
    grid: GridSpec
    mask: CircularMask
    ring: RingGeometry
    cfg: TrainConfig


def small_instance() -> SmallInstance:
    """testsupport::make_small_instance (test_support.hpp:43-75) parameters."""
    cfg = TrainConfig(delays=tuple(make_delays(-0.4, 0.4, 4)), n_angles=32, ray_step=0.1,
                      patch_mm=3.2, overlap=0.0, hidden=8, sine_layers=2, out_scale=60.0,
                      lambda_tv=1e-4, workers=1)
    return SmallInstance(GridSpec.centered(64, 64, 0.1), CircularMask(0.0, 0.0, 2.6),
                         RingGeometry(64, 50.0, 0.0), cfg)
