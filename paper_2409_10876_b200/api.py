"""Python host API over the C-ABI (device-resident, torch tensors as buffers).

Mirrors the reference entry points of the hot path (namespace pact in
/root/reference/proj/include/pact/*.hpp) with the same names and argument
meaning; data lives on the GPU as fp32 torch tensors.  PyTorch is only the
allocator / stream provider here — every computation is a kernel of
libpact_cuda.so (sm_100a).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._abi import Grid, Mask, Ring, SignalMeta, check, darr, dptr


@dataclass(frozen=True)
class RingGeometry:
    """RingGeometry, core.hpp:152-173."""
    n_transducers: int
    radius: float
    angle_offset: float = 0.0

    def c(self) -> Ring:
        return Ring(self.n_transducers, self.radius, self.angle_offset)

    def positions(self) -> np.ndarray:
        a = 2.0 * np.pi * np.arange(self.n_transducers) / self.n_transducers + self.angle_offset
        return np.stack([self.radius * np.cos(a), self.radius * np.sin(a)], axis=1)


@dataclass(frozen=True)
class GridSpec:
    """GridSpec, core.hpp:58-89."""
    width: int
    height: int
    pitch: float
    origin_x: float
    origin_y: float

    @staticmethod
    def centered(width: int, height: int, pitch: float) -> "GridSpec":
        return GridSpec(width, height, pitch, -0.5 * (width - 1) * pitch,
                        -0.5 * (height - 1) * pitch)

    def c(self) -> Grid:
        return Grid(self.width, self.height, self.pitch, self.origin_x, self.origin_y)

    def world(self, ix, iy):
        return self.origin_x + np.asarray(ix) * self.pitch, self.origin_y + np.asarray(iy) * self.pitch


@dataclass(frozen=True)
class SignalMetaInfo:
    """SignalSet scalars, core.hpp:284-313."""
    n_samples: int
    dt: float
    t0: float
    background_sos: float

    def c(self) -> SignalMeta:
        return SignalMeta(self.n_samples, self.dt, self.t0, self.background_sos)


@dataclass(frozen=True)
class CircularMask:
    """CircularMask, core.hpp:175-180."""
    center_x: float
    center_y: float
    radius: float

    def c(self) -> Mask:
        return Mask(self.center_x, self.center_y, self.radius)


def make_delays(lo: float, hi: float, count: int) -> list[float]:
    """make_delays, beamform.hpp:113-120."""
    out = (C.c_double * max(1, count))()
    check(_abi.lib().pact_make_delays(lo, hi, count, out))
    return [out[i] for i in range(count)]


class Context:
    """A pact_ctx bound to a CUDA device, launching on torch's current stream."""

    def __init__(self, device: int = 0):
        self.device = device
        L = _abi.lib()
        h = C.c_void_p()
        torch.cuda.set_device(device)
        check(L.pact_ctx_create(device, C.byref(h)))
        self._h = h
        check(L.pact_ctx_set_stream(self._h, C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))

    def close(self):
        if self._h:
            _abi.lib().pact_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def use_stream(self, stream: torch.cuda.Stream | None):
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        check(_abi.lib().pact_ctx_set_stream(self._h, C.c_void_p(s)))

    def launch_count(self) -> int:
        return int(_abi.lib().pact_ctx_launch_count(self._h))

    # ---- part 1 -----------------------------------------------------------
    def das_stack(self, signals: torch.Tensor, ring: RingGeometry, meta: SignalMetaInfo,
                  grid: GridSpec, v0: float, delays, out: torch.Tensor | None = None) -> torch.Tensor:
        """das_stack, beamform.hpp:77-110 -> fp32 [K, H, W] on the device."""
        assert signals.is_cuda and signals.dtype == torch.float32 and signals.is_contiguous()
        K = len(delays)
        if out is None:
            out = torch.empty((max(K, 1), grid.height, grid.width), device=signals.device,
                              dtype=torch.float32)
        r, m, g = ring.c(), meta.c(), grid.c()
        check(_abi.lib().pact_das_stack(self._h, C.byref(r), C.byref(m), dptr(signals),
                                        C.byref(g), float(v0), darr(delays), K, dptr(out)))
        return out

    def das(self, signals, ring, meta, grid, v0, d):
        """das, beamform.hpp:56-75 (the K = 1 stack)."""
        return self.das_stack(signals, ring, meta, grid, v0, [d])[0]
