"""BASELINE.json configurations (workload_defs.py at the repo root) with the
product's api types, plus the GPU-side fixture helpers (simulate, TrainConfig).

workload_defs.py holds the definitions in pure numpy so that bench.py's
reference arm builds the same workload without loading libpact_cuda.so.
"""
from __future__ import annotations

import os
import sys
from dataclasses import dataclass, fields

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import workload_defs as _d  # noqa: E402
from workload_defs import DT, iid_signals, phantom_rasters, shard_frames  # noqa: E402,F401

from .api import CircularMask, GridSpec, RingGeometry, SignalMetaInfo  # noqa: E402


@dataclass(frozen=True)
class Workload(_d.WorkloadDef):
    @property
    def mask(self) -> CircularMask:
        # D2: "masked to the ring interior" taken literally.
        return CircularMask(0.0, 0.0, self.ring.radius)


def _convert(d: _d.WorkloadDef) -> Workload:
    kw = {f.name: getattr(d, f.name) for f in fields(d)}
    kw["ring"] = RingGeometry(d.ring.n_transducers, d.ring.radius, d.ring.angle_offset)
    kw["meta"] = SignalMetaInfo(d.meta.n_samples, d.meta.dt, d.meta.t0, d.meta.background_sos)
    kw["grid"] = GridSpec(d.grid.width, d.grid.height, d.grid.pitch, d.grid.origin_x,
                          d.grid.origin_y)
    return Workload(**kw)


def cfg1() -> Workload:
    return _convert(_d.cfg1())


def cfg2() -> Workload:
    return _convert(_d.cfg2())


def cfg3() -> Workload:
    return _convert(_d.cfg3())


def cfg5() -> Workload:
    return _convert(_d.cfg5())


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg5": cfg5}


def train_config(w: Workload, **kw):
    """TrainConfig for a workload (Appendix A; reference defaults elsewhere)."""
    from .api import TrainConfig

    return TrainConfig(**_d.train_fields(w, **kw))


def simulation_mask(w: Workload) -> CircularMask:
    """D5: the simulator's TOF disc = image half-diagonal (+ one pitch)."""
    m = _d.simulation_mask(w)
    return CircularMask(m.center_x, m.center_y, m.radius)


def simulate(ctx, w: Workload, seed: int = 0):
    """Signals of the seeded Appendix-A phantom, simulated on the GPU
    (pact_simulate_signals); fp32 [N, T] device tensor."""
    p, sos = phantom_rasters(w, seed)
    return ctx.simulate_signals(w.grid, p, sos, simulation_mask(w), w.v0, w.ring, w.meta)
