"""Helpers to rebuild API objects from golden fixtures."""
import os

import numpy as np

from paper_2409_10876_b200.api import CircularMask, GridSpec, RingGeometry, SignalMetaInfo

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
