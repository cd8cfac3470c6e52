"""BASELINE.json configurations as concrete, seeded synthetic workloads —
pure numpy, with no dependency on the product package, so that bench.py's
reference arm can build the same workload without loading libpact_cuda.so.

The parameter mapping (ring, window, grid, delays, patches, SIREN, mask) is
SURVEY.md Appendix A; where BASELINE.json is silent the reference defaults are
used (optimize.hpp:48-69).  No public dataset is involved: cfg1 signals are
i.i.d. N(0,1); cfg2/3/5 signals are simulated from seeded Gaussian-blob
pressure phantoms and elliptical SOS inclusions (see phantom_rasters()).
The geometry records carry the attribute names of the product's api types
(paper_2409_10876_b200/workloads.py converts them) and of tests/oracle_lib.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DT = 25e-9  # 40 MHz


@dataclass(frozen=True)
class Ring:
    """RingGeometry, core.hpp:152-173."""
    n_transducers: int
    radius: float
    angle_offset: float = 0.0


@dataclass(frozen=True)
class Grid:
    """GridSpec, core.hpp:58-89."""
    width: int
    height: int
    pitch: float
    origin_x: float
    origin_y: float

    @staticmethod
    def centered(width: int, height: int, pitch: float) -> "Grid":
        return Grid(width, height, pitch, -0.5 * (width - 1) * pitch, -0.5 * (height - 1) * pitch)


@dataclass(frozen=True)
class Meta:
    """SignalSet scalars, core.hpp:284-313."""
    n_samples: int
    dt: float
    t0: float
    background_sos: float


@dataclass(frozen=True)
class Mask:
    """CircularMask, core.hpp:175-180."""
    center_x: float
    center_y: float
    radius: float


@dataclass(frozen=True)
class WorkloadDef:
    name: str
    ring: Ring
    meta: Meta
    grid: Grid
    delays: tuple
    v0: float = 1500.0
    patch_mm: float = 0.0
    overlap: float = 0.5
    hidden: int = 64
    sine_layers: int = 3
    omega0: float = 30.0
    out_scale: float = 100.0
    eps_deconv: float = 1e-2
    n_angles: int = 512
    ray_step: float = 0.05
    lambda_tv: float = 3e9
    merge_fwhm: float = 1.5
    n_blobs: int = 0
    n_ellipses: int = 0
    ellipse_sos: tuple = (1540.0, 1580.0)
    extra: dict = field(default_factory=dict)

    @property
    def mask(self) -> Mask:
        # D2: "masked to the ring interior" taken literally.
        return Mask(0.0, 0.0, self.ring.radius)

    @property
    def das_samples(self) -> int:
        """S = W*H*K*N taps of one DAS stack."""
        return self.grid.width * self.grid.height * len(self.delays) * self.ring.n_transducers

    @property
    def das_bytes(self) -> int:
        """Algorithmic bytes of one DAS stack: 8*S + 4*K*W*H + 4*N*T."""
        K, W, H = len(self.delays), self.grid.width, self.grid.height
        return 8 * self.das_samples + 4 * K * W * H + 4 * self.ring.n_transducers * self.meta.n_samples


def _delays(lo, hi, k):
    """make_delays, beamform.hpp:113-120."""
    return tuple(lo + (hi - lo) * j / (k - 1) for j in range(k)) if k > 1 else (lo,)


def _auto_t0(R, grid: Grid, d_max, v_max, sigma=100e-9):
    """Appendix A t0 rule: dt * floor((1e-3 (R - r_max - d_max)/v_max - 8 sigma)/dt)."""
    r_max = math.hypot((grid.width - 1) * grid.pitch / 2, (grid.height - 1) * grid.pitch / 2)
    return DT * math.floor((1e-3 * (R - r_max - d_max) / v_max - 8 * sigma) / DT)


def cfg1() -> WorkloadDef:
    grid = Grid.centered(128, 128, 0.2)
    return WorkloadDef("cfg1", Ring(128, 50.0), Meta(1024, DT, 827 * DT, 1500.0), grid,
                       _delays(-1.0, 1.0, 8))


def cfg2() -> WorkloadDef:
    grid = Grid.centered(256, 256, 0.1)
    t0 = _auto_t0(60.0, grid, 1.5, 1580.0)
    return WorkloadDef("cfg2", Ring(256, 60.0), Meta(2048, DT, t0, 1500.0), grid,
                       _delays(-1.5, 1.5, 16), patch_mm=6.4, overlap=0.5, hidden=64,
                       sine_layers=3, n_blobs=20, n_ellipses=1)


def cfg3() -> WorkloadDef:
    grid = Grid.centered(512, 512, 0.1)
    t0 = _auto_t0(80.0, grid, 2.0, 1580.0)
    return WorkloadDef("cfg3", Ring(512, 80.0), Meta(4096, DT, t0, 1500.0), grid,
                       _delays(-2.0, 2.0, 32), patch_mm=6.4, overlap=0.5, hidden=128,
                       sine_layers=4, n_blobs=40, n_ellipses=2)


def cfg5() -> WorkloadDef:
    grid = Grid.centered(2048, 2048, 0.05)
    t0 = _auto_t0(100.0, grid, 3.0, 1600.0)
    return WorkloadDef("cfg5", Ring(1024, 100.0), Meta(8192, DT, t0, 1500.0), grid,
                       _delays(-3.0, 3.0, 64), patch_mm=6.4, overlap=0.5, hidden=256,
                       sine_layers=4, n_blobs=200, n_ellipses=4, ellipse_sos=(1450.0, 1600.0))


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg5": cfg5}


def iid_signals(w: WorkloadDef, seed: int = 0) -> np.ndarray:
    """cfg1 signals: i.i.d. N(0,1), fp32 [N, T] (rounded to fp32 for both sides)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((w.ring.n_transducers, w.meta.n_samples)).astype(np.float32)


def phantom_rasters(w: WorkloadDef, seed: int = 0):
    """Seeded phantom of Appendix A: (pressure, sos) fp64 rasters on w.grid.

    Ellipses first (pixel-centre inside test), then Gaussian blobs truncated at
    3 sigma: centre U(+-0.4 FOV)^2, sigma U(0.2, 1) mm, amplitude U(0.2, 1).
    """
    rng = np.random.default_rng(seed)
    g = w.grid
    fov = g.width * g.pitch
    xs = g.origin_x + np.arange(g.width) * g.pitch
    ys = g.origin_y + np.arange(g.height) * g.pitch
    X, Y = np.meshgrid(xs, ys)
    sos = np.full((g.height, g.width), w.v0)
    for _ in range(w.n_ellipses):
        cx, cy = rng.uniform(-0.25 * fov, 0.25 * fov, 2)
        a, b = rng.uniform(0.1, 0.3, 2) * fov
        th = rng.uniform(0.0, math.pi)
        v = rng.uniform(*w.ellipse_sos)
        c, s = math.cos(th), math.sin(th)
        u = (X - cx) * c + (Y - cy) * s
        t = -(X - cx) * s + (Y - cy) * c
        sos[(u / a) ** 2 + (t / b) ** 2 <= 1.0] = v
    p = np.zeros((g.height, g.width))
    for _ in range(w.n_blobs):
        cx, cy = rng.uniform(-0.4 * fov, 0.4 * fov, 2)
        sg = rng.uniform(0.2, 1.0)
        amp = rng.uniform(0.2, 1.0)
        # the blob is zero beyond 3 sigma: evaluate it on its bounding box only
        r = 3 * sg
        x0 = max(0, int(math.floor((cx - r - g.origin_x) / g.pitch)))
        x1 = min(g.width, int(math.ceil((cx + r - g.origin_x) / g.pitch)) + 1)
        y0 = max(0, int(math.floor((cy - r - g.origin_y) / g.pitch)))
        y1 = min(g.height, int(math.ceil((cy + r - g.origin_y) / g.pitch)) + 1)
        if x0 >= x1 or y0 >= y1:
            continue
        r2 = (X[y0:y1, x0:x1] - cx) ** 2 + (Y[y0:y1, x0:x1] - cy) ** 2
        blob = amp * np.exp(-0.5 * r2 / sg**2)
        blob[r2 > (3 * sg) ** 2] = 0.0
        p[y0:y1, x0:x1] += blob
    return p, sos


def simulation_mask(w: WorkloadDef) -> Mask:
    """D5: the simulator's TOF disc = image half-diagonal (+ one pitch)."""
    g = w.grid
    return Mask(0.0, 0.0, math.hypot((g.width - 1) * g.pitch / 2, (g.height - 1) * g.pitch / 2)
                + g.pitch)


def train_fields(w: WorkloadDef, **kw) -> dict:
    """TrainConfig fields for a workload (Appendix A; reference defaults
    elsewhere, optimize.hpp:48-69)."""
    d = dict(epochs=10, steps_per_epoch=30, learning_rate=1e-3, beta1=0.9, beta2=0.999,
             adam_eps=1e-8, lambda_tv=w.lambda_tv, delays=tuple(w.delays),
             eps_deconv=w.eps_deconv, n_angles=w.n_angles, ray_step=w.ray_step, seed=0,
             hidden=w.hidden, sine_layers=w.sine_layers, omega0=w.omega0,
             out_scale=w.out_scale, patch_mm=w.patch_mm, overlap=w.overlap,
             merge_fwhm=w.merge_fwhm, implicit_xhat_grad=True, workers=0)
    d.update(kw)
    return d


def shard_frames(n_frames: int, rank: int, world: int) -> list[int]:
    """cfg4 sharding: frame f runs on rank f % world (independent units, no
    data-path collective)."""
    return [f for f in range(n_frames) if f % world == rank]
