"""TEST INFRASTRUCTURE: ctypes view of the CPU oracle builds.

orc = oracle/liboracle.so (the C restatement, oracle/pact_oracle.c)
ref = oracle/_ref/libpact_ref.so (the reference headers compiled in place;
      may be absent on a GPU box without the prebuilt file).
Both export the same signatures with prefixes orc_ / ref_.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORC_PATH = os.path.join(ROOT, "oracle", "liboracle.so")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libpact_ref.so")

_D = C.c_double
_I = C.c_int
_P = C.c_void_p

SIGS = {
    "das_stack": [_I, _D, _D, _I, _D, _D, _P, _I, _I, _D, _D, _D, _D, _I, _P, _I, _P],
}


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        for name, args in SIGS.items():
            fn = getattr(self.lib, prefix + name, None)
            if fn is None:
                continue
            fn.argtypes = args
            fn.restype = C.c_int

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def das_stack(self, sig, ring, meta, grid, v0, delays, workers=0):
        sig = np.ascontiguousarray(sig, dtype=np.float64)
        d = np.ascontiguousarray(delays, dtype=np.float64)
        out = np.zeros((len(d), grid.height, grid.width))
        rc = self.fn("das_stack")(ring.n_transducers, ring.radius, ring.angle_offset,
                                  meta.n_samples, meta.dt, meta.t0, _p(sig), grid.width,
                                  grid.height, grid.pitch, grid.origin_x, grid.origin_y, v0,
                                  len(d), _p(d), workers, _p(out))
        if rc != 0:
            raise RuntimeError(f"{self.prefix}das_stack failed: {rc}")
        return out


_orc = None
_ref = None


def orc() -> Oracle:
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_PATH):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                           capture_output=True)
        _orc = Oracle(ORC_PATH, "orc_")
    return _orc


def ref() -> Oracle | None:
    global _ref
    if _ref is None and os.path.exists(REF_PATH):
        _ref = Oracle(REF_PATH, "ref_")
    return _ref


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128 if np.iscomplexobj(a) else np.float64)
    b = np.asarray(b, dtype=a.dtype)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den > 0 else 1.0))
