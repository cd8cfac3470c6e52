"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref).

Run in the build container (where /root/reference is mounted and
oracle/_ref/libpact_ref.so was compiled from it):
    python tests/golden/make_golden.py
Every fixture stores its inputs (already rounded to fp32 where the GPU path
consumes fp32) and the reference outputs in fp64.  The GPU box never needs
/root/reference: the tests read these files.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import ref  # noqa: E402
from paper_2409_10876_b200 import workloads as wl  # noqa: E402
from paper_2409_10876_b200.api import GridSpec, RingGeometry, SignalMetaInfo  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes raw")


def grid_arr(g: GridSpec):
    return np.array([g.width, g.height, g.pitch, g.origin_x, g.origin_y])


def ring_arr(r: RingGeometry):
    return np.array([r.n_transducers, r.radius, r.angle_offset])


def meta_arr(m: SignalMetaInfo):
    return np.array([m.n_samples, m.dt, m.t0, m.background_sos])


def das_cases(R):
    rng = np.random.default_rng(1234)
    # (a) small non-square grid with a clipped time window: many taps fall
    # outside [0, T-1] and exercise SignalSet::sample edge semantics.
    ring = RingGeometry(32, 30.0, 0.1)
    meta = SignalMetaInfo(160, 25e-9, 19.0e-6, 1500.0)
    grid = GridSpec(24, 20, 0.25, -2.9, -2.2)
    sig = rng.standard_normal((32, 160)).astype(np.float32).astype(np.float64)
    delays = np.array([-1.0, -0.35, 0.2, 0.9, 1.5])
    out = R.das_stack(sig, ring, meta, grid, 1500.0, delays, workers=1)
    save("das_edge", ring=ring_arr(ring), meta=meta_arr(meta), grid=grid_arr(grid), sig=sig,
         delays=delays, v0=np.array(1500.0), out=out)

    # (b) cfg1 geometry (BASELINE configs[0]) on a 32x32 crop of the 128x128
    # grid; signals are the cfg1 i.i.d. N(0,1) draw (seed 0), stored.
    w = wl.cfg1()
    sig1 = wl.iid_signals(w, 0).astype(np.float64)
    g = w.grid
    crop = GridSpec(32, 32, g.pitch, g.origin_x + 40 * g.pitch, g.origin_y + 70 * g.pitch)
    out1 = R.das_stack(sig1, w.ring, w.meta, crop, w.v0, np.array(w.delays), workers=0)
    save("das_cfg1_crop", ring=ring_arr(w.ring), meta=meta_arr(w.meta), grid=grid_arr(crop),
         sig=sig1.astype(np.float32), delays=np.array(w.delays), v0=np.array(w.v0), out=out1)


def main():
    R = ref()
    if R is None:
        sys.exit("oracle/_ref/libpact_ref.so missing: make -C oracle ref")
    das_cases(R)


if __name__ == "__main__":
    main()
