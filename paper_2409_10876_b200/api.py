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


@dataclass(frozen=True)
class BodyModel:
    """BodyModel, beamform.hpp:44-54."""
    center_x: float
    center_y: float
    radius: float
    body_sos: float

    def c(self) -> "_abi.Body":
        return _abi.Body(self.center_x, self.center_y, self.radius, self.body_sos)


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

    # ---- multi-GPU frame over NCCL (pact_ctx owns the communicator) -------
    @staticmethod
    def nccl_unique_id() -> bytes:
        """pact_nccl_unique_id: rank 0 makes it, every rank attaches it."""
        buf = (C.c_ubyte * 128)()
        check(_abi.lib().pact_nccl_unique_id(buf))
        return bytes(buf)

    def attach_nccl(self, uid: bytes, rank: int, world: int):
        """pact_ctx_attach_nccl: ncclCommInitRank on this context's device."""
        assert len(uid) == 128
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        check(_abi.lib().pact_ctx_attach_nccl(self._h, buf, int(rank), int(world)))

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

    def dual_sos_das(self, signals: torch.Tensor, ring: RingGeometry, meta: SignalMetaInfo,
                     grid: GridSpec, v0: float, body: "BodyModel",
                     out: torch.Tensor | None = None) -> torch.Tensor:
        """dual_sos_das, beamform.hpp:124-150 -> fp32 [H, W] on the device."""
        assert signals.is_cuda and signals.dtype == torch.float32 and signals.is_contiguous()
        if out is None:
            out = torch.empty((grid.height, grid.width), device=signals.device, dtype=torch.float32)
        r, m, g, b = ring.c(), meta.c(), grid.c(), body.c()
        check(_abi.lib().pact_dual_sos_das(self._h, C.byref(r), C.byref(m), dptr(signals),
                                           C.byref(g), float(v0), C.byref(b), dptr(out)))
        return out


# --------------------------------------------------------------------------- #
# patch layout, SIREN, PSF, deconvolution, loss and gradients
# --------------------------------------------------------------------------- #

@dataclass(frozen=True)
class PatchLayout:
    """PatchLayout, core.hpp:222-281 (built by make_patch_layout)."""
    raw: object
    offsets: np.ndarray  # [n, 2] (ox, oy)
    centers: np.ndarray  # [n, 2] world mm

    @property
    def patch_pixels(self) -> int:
        return self.raw.patch_pixels

    @property
    def n_patches(self) -> int:
        return self.raw.nx * self.raw.ny

    def c(self):
        return self.raw


def make_patch_layout(grid: GridSpec, patch_mm: float, overlap: float) -> PatchLayout:
    """make_patch_layout, core.hpp:252-281."""
    L = _abi.lib()
    lay = _abi.Layout()
    g = grid.c()
    check(L.pact_make_patch_layout(C.byref(g), patch_mm, overlap, C.byref(lay)))
    n = lay.nx * lay.ny
    off = np.zeros((n, 2), np.int32)
    cen = np.zeros((n, 2), np.float64)
    check(L.pact_layout_patches(C.byref(lay), off.ctypes.data_as(C.POINTER(C.c_int32)),
                                cen.ctypes.data_as(C.POINTER(C.c_double))))
    return PatchLayout(lay, off, cen)


@dataclass(frozen=True)
class SirenSpec:
    """SirenParams scalars, nfield.hpp:37-71."""
    hidden: int = 64
    n_hidden_layers: int = 2
    omega0: float = 30.0
    out_scale: float = 100.0
    v0: float = 1500.0

    def c(self):
        return _abi.Siren(2, self.hidden, self.n_hidden_layers, self.omega0, self.out_scale,
                          self.v0)

    def param_count(self) -> int:
        s = self.c()
        return int(_abi.lib().pact_siren_param_count(C.byref(s)))


def init_siren(seed: int, spec: SirenSpec) -> np.ndarray:
    """init_siren, nfield.hpp:83-107 (fp64, bit-identical to the reference)."""
    th = np.zeros(spec.param_count(), np.float64)
    s = spec.c()
    check(_abi.lib().pact_init_siren(seed, C.byref(s), th.ctypes.data_as(C.POINTER(C.c_double))))
    return th


def masked_pixels(grid: GridSpec, mask: CircularMask):
    """render_sos's masked pixel list: (flat indices, normalised coords)."""
    L = _abi.lib()
    g, m = grid.c(), mask.c()
    n = L.pact_masked_count(C.byref(g), C.byref(m))
    idx = np.zeros(max(n, 1), np.int32)
    co = np.zeros((max(n, 1), 2), np.float32)
    check(L.pact_masked_pixels(C.byref(g), C.byref(m), idx.ctypes.data_as(C.POINTER(C.c_int32)),
                               co.ctypes.data_as(C.POINTER(C.c_float))))
    return idx[:n], co[:n]


@dataclass(frozen=True)
class DeconvolveOptions:
    """DeconvolveOptions, deconv.hpp:166-172."""
    eps: float = 1e-3
    n_angles: int = 512
    ray_step: float = 0.05
    merge_fwhm: float = 1.5

    def c(self):
        return _abi.DeconvOptions(self.eps, self.n_angles, self.ray_step, self.merge_fwhm)


def _cplx(t: torch.Tensor) -> torch.Tensor:
    return t if t.dtype == torch.complex64 else t.to(torch.complex64)


def _need(t, name: str, dtype, numel: int | None = None) -> torch.Tensor:
    """Argument check before a raw device pointer crosses the C-ABI: CUDA,
    the expected dtype and (optionally) element count; returns it contiguous."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError(f"{name}: CUDA tensor expected")
    if t.dtype != dtype:
        raise TypeError(f"{name}: {dtype} expected, got {t.dtype}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name}: {numel} elements expected, got {t.numel()}")
    return t.contiguous()


def _ctx_methods():
    def render_sos(self, spec: SirenSpec, theta: torch.Tensor, grid: GridSpec,
                   mask: CircularMask):
        """render_sos, nfield.hpp:145-162 -> (raster v, deviation v - v0), fp32 [H, W]."""
        theta = theta.to(device="cuda", dtype=torch.float32).contiguous()
        raster = torch.empty((grid.height, grid.width), device="cuda", dtype=torch.float32)
        dev = torch.empty_like(raster)
        s, g, m = spec.c(), grid.c(), mask.c()
        check(_abi.lib().pact_render_sos(self._h, C.byref(s), dptr(theta), C.byref(g), C.byref(m),
                                         dptr(raster), dptr(dev)))
        return raster, dev

    def siren_backward(self, spec: SirenSpec, theta: torch.Tensor, grid: GridSpec,
                       mask: CircularMask, grad_masked: torch.Tensor) -> torch.Tensor:
        """backprop_sos, nfield.hpp:166-233 -> fp64 [param_count]."""
        theta = theta.to(device="cuda", dtype=torch.float32).contiguous()
        gm = grad_masked.to(device="cuda", dtype=torch.float32).contiguous()
        out = torch.empty(spec.param_count(), device="cuda", dtype=torch.float64)
        s, g, m = spec.c(), grid.c(), mask.c()
        check(_abi.lib().pact_siren_backward(self._h, C.byref(s), dptr(theta), C.byref(g),
                                             C.byref(m), dptr(gm), dptr(out)))
        return out

    def wavefront(self, ring: RingGeometry, grid: GridSpec, sos_dev: torch.Tensor, v0: float,
                  mask: CircularMask, centers, n_angles: int, step: float) -> torch.Tensor:
        """wavefront_profile, aberration.hpp:134-186 for every centre -> fp32 [n, A]."""
        cen = np.ascontiguousarray(np.asarray(centers, np.float64).reshape(-1, 2))
        n = cen.shape[0]
        sos_dev = _need(sos_dev, "sos_dev", torch.float32, grid.width * grid.height)
        w = torch.empty((n, n_angles), device="cuda", dtype=torch.float32)
        r, g, m = ring.c(), grid.c(), mask.c()
        check(_abi.lib().pact_wavefront(self._h, C.byref(r), C.byref(g), dptr(sos_dev),
                                        v0, C.byref(m), n,
                                        cen.ctypes.data_as(C.POINTER(C.c_double)), n_angles, step,
                                        dptr(w)))
        return w

    def transfer_stack(self, w: torch.Tensor, delays, P: int, pitch: float) -> torch.Tensor:
        """transfer_stack, aberration.hpp:236-265 -> complex64 [n, K, P, P]."""
        w = _need(w, "w", torch.float32)
        n, A = w.shape
        K = len(delays)
        H = torch.empty((n, K, P, P), device="cuda", dtype=torch.complex64)
        check(_abi.lib().pact_transfer_stack(self._h, n, dptr(w), A, darr(delays), K, P, pitch,
                                             dptr(H)))
        return H

    def patch_spectra(self, layout: PatchLayout, stack: torch.Tensor) -> torch.Tensor:
        """extract_patch_spectra, deconv.hpp:64-74 -> complex64 [n, K, P, P]."""
        g = layout.raw.grid
        stack = _need(stack, "stack", torch.float32)
        if stack.dim() != 3 or stack.shape[1:] != (g.height, g.width):
            raise ValueError("stack: [K, H, W] on the layout grid expected")
        K = stack.shape[0]
        P = layout.patch_pixels
        Y = torch.empty((layout.n_patches, K, P, P), device="cuda", dtype=torch.complex64)
        lay = layout.c()
        check(_abi.lib().pact_patch_spectra(self._h, C.byref(lay), dptr(stack.contiguous()), K,
                                            dptr(Y)))
        return Y

    def deconvolve_image(self, stack: torch.Tensor, delays, v0: float, sos_dev: torch.Tensor,
                         ring: RingGeometry, mask: CircularMask, layout: PatchLayout,
                         opt: DeconvolveOptions) -> torch.Tensor:
        """deconvolve_image, deconv.hpp:176-198 -> fp32 [H, W]."""
        g = layout.raw.grid
        stack = _need(stack, "stack", torch.float32, len(delays) * g.height * g.width)
        sos_dev = _need(sos_dev, "sos_dev", torch.float32, g.height * g.width)
        img = torch.empty((g.height, g.width), device="cuda", dtype=torch.float32)
        r, m, lay, o = ring.c(), mask.c(), layout.c(), opt.c()
        check(_abi.lib().pact_deconvolve_image(self._h, dptr(stack.contiguous()), len(delays),
                                               darr(delays), v0, dptr(sos_dev.contiguous()),
                                               C.byref(r), C.byref(m), C.byref(lay), C.byref(o),
                                               dptr(img)))
        return img

    def loss_grad(self, Y: torch.Tensor, w: torch.Tensor, delays, P: int, pitch: float,
                  eps: float, scale: float, implicit: bool = True):
        """fused_patch_loss_grad, optimize.hpp:234-325, batched -> (loss fp64 [n], dw fp32 [n, A])."""
        w = _need(w, "w", torch.float32)
        n, A = w.shape
        Y = _need(_cplx(Y), "Y", torch.complex64, n * len(delays) * P * P)
        loss = torch.empty(n, device="cuda", dtype=torch.float64)
        dw = torch.empty_like(w)
        check(_abi.lib().pact_loss_grad(self._h, n, dptr(Y), dptr(w), A, darr(delays), len(delays),
                                        P, pitch, eps, scale, 1 if implicit else 0, dptr(loss),
                                        dptr(dw)))
        return loss, dw

    def ray_backward(self, ring: RingGeometry, grid: GridSpec, sos_dev: torch.Tensor, v0: float,
                     mask: CircularMask, centers, n_angles: int, step: float, dw: torch.Tensor,
                     grad_v: torch.Tensor | None = None) -> torch.Tensor:
        """wavefront_grad_trace, aberration.hpp:333-361, batched: grad_v (fp64 [H, W]) +=."""
        cen = np.ascontiguousarray(np.asarray(centers, np.float64).reshape(-1, 2))
        if grad_v is None:
            grad_v = torch.zeros((grid.height, grid.width), device="cuda", dtype=torch.float64)
        _need(grad_v, "grad_v", torch.float64, grid.height * grid.width)
        assert grad_v.is_contiguous(), "grad_v: contiguous fp64 accumulator expected"
        sos_dev = _need(sos_dev, "sos_dev", torch.float32, grid.height * grid.width)
        dw = _need(dw, "dw", torch.float32, cen.shape[0] * n_angles)
        r, g, m = ring.c(), grid.c(), mask.c()
        check(_abi.lib().pact_ray_backward(self._h, C.byref(r), C.byref(g),
                                           dptr(sos_dev), v0, C.byref(m),
                                           cen.shape[0], cen.ctypes.data_as(C.POINTER(C.c_double)),
                                           n_angles, step, dptr(dw), dptr(grad_v)))
        return grad_v

    def tv_loss(self, grid: GridSpec, mask: CircularMask, raster: torch.Tensor, lam: float):
        """tv_loss, optimize.hpp:120-153 -> (value, grad per masked pixel fp32)."""
        g, m = grid.c(), mask.c()
        n = _abi.lib().pact_masked_count(C.byref(g), C.byref(m))
        grad = torch.empty(max(n, 1), device="cuda", dtype=torch.float32)
        val = C.c_double()
        check(_abi.lib().pact_tv_loss(self._h, C.byref(g), C.byref(m), dptr(raster.contiguous()),
                                      lam, C.byref(val), dptr(grad)))
        return val.value, grad[:n]

    def adam_step(self, theta, grad, m, v, t, lr, beta1, beta2, eps):
        """adam_step, optimize.hpp:87-110 on fp64 device tensors (t after the update)."""
        n = theta.numel()
        for name, t in (("theta", theta), ("grad", grad), ("m", m), ("v", v)):
            _need(t, name, torch.float64, n)
            assert t.is_contiguous(), f"{name}: contiguous tensor expected"
        check(_abi.lib().pact_adam_step(self._h, theta.numel(), dptr(theta), dptr(grad), dptr(m),
                                        dptr(v), t, lr, beta1, beta2, eps))

    def simulate_signals(self, grid: GridSpec, pressure, sos, mask: CircularMask,
                         background_sos: float, ring: RingGeometry, meta: SignalMetaInfo,
                         pulse_sigma: float = 100e-9, ray_step: float = 0.05,
                         spreading: bool = False) -> torch.Tensor:
        """simulate_signals, phantom.hpp:282-362 -> fp32 [N, T] on the device
        (`spreading`: SimulateOptions::spreading, amplitude / sqrt(distance))."""
        pr = np.ascontiguousarray(pressure, np.float64)
        so = np.ascontiguousarray(sos, np.float64)
        out = torch.empty((ring.n_transducers, meta.n_samples), device="cuda", dtype=torch.float32)
        g, m, r, mt = grid.c(), mask.c(), ring.c(), meta.c()
        check(_abi.lib().pact_simulate_signals_ex(self._h, C.byref(g),
                                                  pr.ctypes.data_as(C.POINTER(C.c_double)),
                                                  so.ctypes.data_as(C.POINTER(C.c_double)),
                                                  C.byref(m), background_sos, C.byref(r),
                                                  pulse_sigma, C.byref(mt), ray_step,
                                                  1 if spreading else 0, dptr(out)))
        return out

    # ---- the composed (non-fused) path, fp64 (composed.cu) ----
    def _c128(t, name, ndim):
        assert isinstance(t, torch.Tensor) and t.is_cuda, f"{name}: CUDA tensor expected"
        assert t.dtype == torch.complex128 and t.dim() == ndim, \
            f"{name}: complex128 tensor with {ndim} dims expected"
        return t.contiguous()

    def multichannel_deconvolve(self, Y: torch.Tensor, H: torch.Tensor, eps: float) -> torch.Tensor:
        """multichannel_deconvolve, deconv.hpp:78-96, batched: complex128
        [n, K, P, P] x2 -> X complex128 [n, P, P]."""
        Y, H = _c128(Y, "Y", 4), _c128(H, "H", 4)
        if Y.shape != H.shape:
            raise _abi.ValidationError(2, "deconvolve: Y and H channel counts differ")
        n, K, P, _ = Y.shape
        X = torch.empty((n, P, P), device="cuda", dtype=torch.complex128)
        check(_abi.lib().pact_multichannel_deconvolve(self._h, n, K, P, dptr(Y), dptr(H), eps,
                                                      dptr(X)))
        return X

    def deconv_jacobian_H(self, Y: torch.Tensor, H: torch.Tensor, eps: float, queries):
        """deconv_jacobian_H, deconv.hpp:100-115 for queries [(patch, j, bin)]
        -> complex128 [q, 2] = (dX/dRe H_j, dX/dIm H_j) at the bin."""
        Y, H = _c128(Y, "Y", 4), _c128(H, "H", 4)
        n, K, P, _ = Y.shape
        q = torch.as_tensor(np.asarray(queries, np.int32).reshape(-1, 3)).cuda()
        out = torch.empty((q.shape[0], 2), device="cuda", dtype=torch.complex128)
        check(_abi.lib().pact_deconv_jacobian_H(self._h, K, P, dptr(Y), dptr(H), eps, q.shape[0],
                                                dptr(q), dptr(out)))
        torch.cuda.current_stream().synchronize()
        return out

    def patch_data_loss(self, Y: torch.Tensor, H: torch.Tensor, pitch: float, eps: float,
                        scale: float, implicit: bool = True):
        """patch_data_loss, optimize.hpp:164-211, batched -> (loss fp64 [n],
        grad_h complex128 [n, K, P, P])."""
        Y, H = _c128(Y, "Y", 4), _c128(H, "H", 4)
        if Y.shape != H.shape:
            raise _abi.ValidationError(2, "data_loss: Y/H channel mismatch")
        n, K, P, _ = Y.shape
        loss = torch.empty(n, device="cuda", dtype=torch.float64)
        g = torch.empty_like(Y)
        check(_abi.lib().pact_patch_data_loss(self._h, n, K, P, pitch, dptr(Y), dptr(H), eps, scale,
                                              1 if implicit else 0, dptr(loss), dptr(g)))
        return loss, g

    def data_loss(self, Y: torch.Tensor, H: torch.Tensor, pitch: float, eps: float,
                  implicit: bool = True):
        """data_loss, optimize.hpp:336-353 -> (value, loss fp64 [n], grad_h)."""
        Y, H = _c128(Y, "Y", 4), _c128(H, "H", 4)
        if Y.shape[0] != H.shape[0]:
            raise _abi.ValidationError(2, "data_loss: patch count mismatch")
        if Y.shape != H.shape:
            raise _abi.ValidationError(2, "data_loss: Y/H channel mismatch")
        n, K, P, _ = Y.shape
        loss = torch.empty(n, device="cuda", dtype=torch.float64)
        g = torch.empty_like(Y)
        val = C.c_double()
        check(_abi.lib().pact_data_loss(self._h, n, K, P, pitch, dptr(Y), dptr(H), eps,
                                        1 if implicit else 0, C.byref(val), dptr(loss), dptr(g)))
        return val.value, loss, g

    def transfer_grad_to_wavefront(self, w: torch.Tensor, delays, P: int, pitch: float,
                                   grad_h: torch.Tensor) -> torch.Tensor:
        """transfer_grad_to_wavefront, aberration.hpp:270-313, batched:
        w fp64 [n, A], grad_h complex128 [n, K, P, P] -> dw fp64 [n, A]."""
        assert w.is_cuda and w.dtype == torch.float64 and w.dim() == 2, "w: CUDA fp64 [n, A]"
        g = _c128(grad_h, "grad_h", 4)
        n, A = w.shape
        assert g.shape == (n, len(delays), P, P), "grad_h: [n, K, P, P] expected"
        dw = torch.empty_like(w)
        check(_abi.lib().pact_transfer_grad_to_wavefront(self._h, n, dptr(w.contiguous()), A,
                                                         darr(delays), len(delays), P, pitch,
                                                         dptr(g), dptr(dw)))
        return dw

    def wavefront_jacobian(self, ring: RingGeometry, grid: GridSpec, sos_dev: torch.Tensor,
                           v0: float, mask: CircularMask, centers, n_angles: int, step: float):
        """wavefront_profile(..., with_jacobian=true), aberration.hpp:134-186 ->
        (w fp64 [n, A], row_start int64 [n A + 1], pixel int32 [nnz], dw_dv fp32 [nnz])."""
        assert sos_dev.is_cuda and sos_dev.dtype == torch.float32, "sos_dev: CUDA fp32 [H, W]"
        assert sos_dev.numel() == grid.width * grid.height, "sos_dev: grid-sized raster expected"
        cen = np.ascontiguousarray(np.asarray(centers, np.float64).reshape(-1, 2))
        n = cen.shape[0]
        w = torch.empty((n, n_angles), device="cuda", dtype=torch.float64)
        rs = torch.empty(n * n_angles + 1, device="cuda", dtype=torch.int64)
        nnz = C.c_int64()
        r, g, m = ring.c(), grid.c(), mask.c()
        cp = cen.ctypes.data_as(C.POINTER(C.c_double))
        L = _abi.lib()
        sd = dptr(sos_dev.contiguous())
        check(L.pact_wavefront_jacobian(self._h, C.byref(r), C.byref(g), sd, v0, C.byref(m), n, cp,
                                        n_angles, step, None, dptr(rs), None, None, 0,
                                        C.byref(nnz)))
        pix = torch.empty(max(nnz.value, 1), device="cuda", dtype=torch.int32)
        val = torch.empty(max(nnz.value, 1), device="cuda", dtype=torch.float32)
        check(L.pact_wavefront_jacobian(self._h, C.byref(r), C.byref(g), sd, v0, C.byref(m), n, cp,
                                        n_angles, step, dptr(w), dptr(rs), dptr(pix), dptr(val),
                                        pix.numel(), C.byref(nnz)))
        return w, rs, pix[:nnz.value], val[:nnz.value]

    def accumulate_wavefront_grad(self, row_start: torch.Tensor, pixel: torch.Tensor,
                                  dw_dv: torch.Tensor, dw: torch.Tensor, grad_v: torch.Tensor):
        """accumulate_wavefront_grad, aberration.hpp:316-326: grad_v (fp64) += J^T dw."""
        assert grad_v.is_cuda and grad_v.dtype == torch.float64, "grad_v: CUDA fp64"
        assert dw.is_cuda and dw.dtype == torch.float64, "dw: CUDA fp64"
        n_rows = row_start.numel() - 1
        assert dw.numel() == n_rows, "dw: one value per Jacobian row"
        check(_abi.lib().pact_accumulate_wavefront_grad(self._h, n_rows, dptr(row_start),
                                                        dptr(pixel), dptr(dw_dv),
                                                        dptr(dw.contiguous()), dptr(grad_v)))
        return grad_v

    def psf_from_transfer(self, spectra: torch.Tensor) -> torch.Tensor:
        """psf_from_transfer, aberration.hpp:407-445, batched (fp64): complex128
        [n, P, P] conjugate-symmetric spectra -> centred real PSFs fp64 [n, P, P]
        (zero lag at (P/2, P/2); the raster origin is -(P/2) pitch)."""
        S = _c128(spectra, "spectra", 3)
        n, P, _ = S.shape
        out = torch.empty((n, P, P), device="cuda", dtype=torch.float64)
        check(_abi.lib().pact_psf_from_transfer(self._h, n, P, dptr(S), dptr(out)))
        return out

    def merge_patches(self, layout: PatchLayout, patches: torch.Tensor, fwhm: float) -> torch.Tensor:
        """merge_patches + MergeWindow, deconv.hpp:118-164: fp32 [n, P, P] -> fp32 [H, W]."""
        P = layout.patch_pixels
        if patches.shape != (layout.n_patches, P, P):
            raise _abi.ValidationError(2, "merge_patches: patch count does not match layout")
        assert patches.is_cuda and patches.dtype == torch.float32, "patches: CUDA fp32"
        g = layout.raw.grid
        img = torch.empty((g.height, g.width), device="cuda", dtype=torch.float32)
        lay = layout.c()
        check(_abi.lib().pact_merge_patches(self._h, C.byref(lay), dptr(patches.contiguous()), None,
                                            fwhm, dptr(img)))
        return img

    for f in (simulate_signals, render_sos, siren_backward, wavefront, transfer_stack, patch_spectra,
              deconvolve_image, loss_grad, ray_backward, tv_loss, adam_step,
              multichannel_deconvolve, deconv_jacobian_H, patch_data_loss, data_loss,
              transfer_grad_to_wavefront, wavefront_jacobian, accumulate_wavefront_grad,
              merge_patches, psf_from_transfer):
        setattr(Context, f.__name__, f)


_ctx_methods()


def simulate_window(grid: GridSpec, pressure, sos, background_sos: float, ring: RingGeometry,
                    pulse_sigma: float = 100e-9, dt: float = 25e-9, t0: float = float("nan"),
                    n_samples: int = 0) -> SignalMetaInfo:
    """The acquisition window of simulate_signals (phantom.hpp:284-334), host only:
    t0 = NaN / n_samples = 0 select the automatic window."""
    pr = np.ascontiguousarray(pressure, np.float64)
    so = np.ascontiguousarray(sos, np.float64)
    g, r, out = grid.c(), ring.c(), _abi.SignalMeta()
    check(_abi.lib().pact_simulate_window(C.byref(g), pr.ctypes.data_as(C.POINTER(C.c_double)),
                                          so.ctypes.data_as(C.POINTER(C.c_double)),
                                          background_sos, C.byref(r), pulse_sigma, dt, t0,
                                          n_samples, C.byref(out)))
    return SignalMetaInfo(out.n_samples, out.dt, out.t0, out.background_sos)


# --------------------------------------------------------------------------- #
# joint_reconstruct engine
# --------------------------------------------------------------------------- #

@dataclass
class TrainConfig:
    """TrainConfig, optimize.hpp:48-78 (reference defaults)."""
    epochs: int = 10
    steps_per_epoch: int = 30
    learning_rate: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    lambda_tv: float = 3e9
    delays: tuple = tuple(-0.8 + 1.6 * j / 31 for j in range(32))
    eps_deconv: float = 1e-3
    n_angles: int = 512
    ray_step: float = 0.05
    seed: int = 0
    hidden: int = 64
    sine_layers: int = 2
    omega0: float = 30.0
    out_scale: float = 100.0
    patch_mm: float = 3.2
    overlap: float = 0.75
    merge_fwhm: float = 1.5
    implicit_xhat_grad: bool = True
    workers: int = 0
    use_cuda_graph: bool = True

    def c(self):
        arr = (C.c_double * len(self.delays))(*[float(d) for d in self.delays])
        cfg = _abi.TrainConfig(self.epochs, self.steps_per_epoch, self.learning_rate, self.beta1,
                               self.beta2, self.adam_eps, self.lambda_tv, len(self.delays),
                               C.cast(arr, C.POINTER(C.c_double)), self.eps_deconv, self.n_angles,
                               self.ray_step, self.seed, self.hidden, self.sine_layers,
                               self.omega0, self.out_scale, self.patch_mm, self.overlap,
                               self.merge_fwhm, 1 if self.implicit_xhat_grad else 0, self.workers,
                               1 if self.use_cuda_graph else 0)
        return cfg, arr


_TORCH_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4",
                  torch.complex64: "<c8", torch.uint8: "|u1"}


def _device_view(ptr: int, shape, dtype: torch.dtype) -> torch.Tensor:
    """torch tensor over library-owned device memory (no copy)."""
    class _Iface:
        __cuda_array_interface__ = {"shape": tuple(int(s) for s in shape),
                                    "typestr": _TORCH_TYPESTR[dtype], "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Iface(), device="cuda")


class Trainer:
    """pact_trainer: joint_reconstruct (optimize.hpp:367-494) split into
    create / step / report / finish so the iteration can be timed."""

    def __init__(self, ctx: Context, signals: torch.Tensor, ring: RingGeometry,
                 meta: SignalMetaInfo, grid: GridSpec, mask: CircularMask, cfg: TrainConfig,
                 partition: tuple[int, int] | None = None):
        """partition = (rank, world): this trainer owns a share of one frame and
        steps by phases (see pact_trainer_create_partitioned, distributed.py)."""
        self.ctx, self.grid, self.cfg = ctx, grid, cfg
        self.v0 = meta.background_sos
        self._signals = signals.contiguous()
        c, self._arr = cfg.c()
        r, m, g, mk = ring.c(), meta.c(), grid.c(), mask.c()
        h = C.c_void_p()
        if partition is None:
            check(_abi.lib().pact_trainer_create(ctx.handle, C.byref(r), C.byref(m),
                                                 dptr(self._signals), C.byref(g), C.byref(mk),
                                                 C.byref(c), C.byref(h)))
        else:
            p = _abi.Partition(int(partition[0]), int(partition[1]))
            check(_abi.lib().pact_trainer_create_partitioned(
                ctx.handle, C.byref(r), C.byref(m), dptr(self._signals), C.byref(g), C.byref(mk),
                C.byref(c), C.byref(p), C.byref(h)))
        self._h = h
        self.mask = mask
        self.n_masked = int(_abi.lib().pact_masked_count(C.byref(g), C.byref(mk)))
        self.n_params = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale,
                                  meta.background_sos).param_count()

    def step(self, n: int = 1):
        check(_abi.lib().pact_trainer_step(self._h, n))

    def report(self, epoch: int = 1):
        rep = (C.c_double * 3)()
        check(_abi.lib().pact_trainer_report(self._h, epoch, rep))
        return list(rep)

    def run_epoch(self, epoch: int):
        rep = (C.c_double * 4)()
        check(_abi.lib().pact_trainer_run_epoch(self._h, epoch, rep))
        return list(rep)

    def finish(self):
        img = torch.empty((self.grid.height, self.grid.width), device="cuda", dtype=torch.float32)
        sos = torch.empty_like(img)
        check(_abi.lib().pact_trainer_finish(self._h, dptr(img), dptr(sos)))
        return img, sos

    def theta(self) -> np.ndarray:
        th = np.zeros(self.n_params, np.float64)
        check(_abi.lib().pact_trainer_get_theta(self._h, th.ctypes.data_as(C.POINTER(C.c_double))))
        return th

    def set_theta(self, th: np.ndarray):
        th = np.ascontiguousarray(th, np.float64)
        check(_abi.lib().pact_trainer_set_theta(self._h, th.ctypes.data_as(C.POINTER(C.c_double))))

    def buffer(self, what: int) -> int:
        return int(_abi.lib().pact_trainer_buffer(self._h, what) or 0)

    def phase(self, k: int):
        """pact_trainer_phase: one phase of the iteration (0-3; 1 = 6 then 7)
        or of the final image (4-5); asynchronous on the engine stream."""
        check(_abi.lib().pact_trainer_phase(self._h, int(k)))

    def step_nccl(self, n: int = 1):
        """pact_trainer_step_nccl: n iterations of a partitioned trainer with the
        collectives over the NCCL communicator attached to its context
        (Context.attach_nccl); no host framework involved."""
        check(_abi.lib().pact_trainer_step_nccl(self._h, int(n)))

    def finish_nccl(self):
        """pact_trainer_finish_nccl: the whole frame's image and SOS on every rank."""
        img = torch.empty((self.grid.height, self.grid.width), device="cuda", dtype=torch.float32)
        sos = torch.empty_like(img)
        check(_abi.lib().pact_trainer_finish_nccl(self._h, dptr(img), dptr(sos)))
        return img, sos

    def local(self) -> dict:
        """The partition this trainer owns (pact_trainer_local)."""
        info = (C.c_int32 * 9)()
        check(_abi.lib().pact_trainer_local(self._h, info))
        keys = ("patch_lo", "patch_hi", "pixel_lo", "pixel_hi", "n_patches", "rank", "world",
                "stack_row0", "stack_rows")
        return dict(zip(keys, list(info)))

    def view(self, what: int, shape, dtype: torch.dtype) -> torch.Tensor:
        """A zero-copy torch view of an engine buffer (see pact_trainer_buffer)."""
        return _device_view(self.buffer(what), shape, dtype)

    def read(self, what: int, shape, dtype) -> np.ndarray:
        """Copy an engine buffer (see pact_trainer_buffer) to the host."""
        out = np.zeros(shape, dtype)
        self.stream().synchronize()
        check(_abi.lib().pact_download(self.ctx.handle, C.c_void_p(out.ctypes.data),
                                       C.c_void_p(self.buffer(what)), out.nbytes))
        return out

    def launch_count(self) -> int:
        return int(_abi.lib().pact_trainer_launch_count(self._h))

    def stream(self) -> torch.cuda.ExternalStream:
        """The engine's private CUDA stream (for event timing)."""
        return torch.cuda.ExternalStream(int(_abi.lib().pact_trainer_stream(self._h)))

    STAGES = ("siren_fwd", "wavefront", "fused_loss", "ray_backward", "tv_report", "siren_bwd",
              "adam")

    def profile_step(self) -> dict:
        """One iteration with CUDA events between stages -> {stage: ms}."""
        ms = (C.c_float * 7)()
        check(_abi.lib().pact_trainer_profile_step(self._h, ms))
        return dict(zip(self.STAGES, [float(x) for x in ms]))

    def close(self):
        if self._h:
            _abi.lib().pact_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def joint_reconstruct(ctx: Context, signals: torch.Tensor, ring: RingGeometry,
                      meta: SignalMetaInfo, grid: GridSpec, mask: CircularMask, cfg: TrainConfig):
    """joint_reconstruct, optimize.hpp:367-494 -> (reports [epochs, 4], image, sos, theta)."""
    c, arr = cfg.c()
    reps = np.zeros((cfg.epochs, 4))
    img = torch.empty((grid.height, grid.width), device="cuda", dtype=torch.float32)
    sos = torch.empty_like(img)
    n = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale,
                  meta.background_sos).param_count()
    th = np.zeros(n, np.float64)
    r, m, g, mk = ring.c(), meta.c(), grid.c(), mask.c()
    check(_abi.lib().pact_joint_reconstruct(ctx.handle, C.byref(r), C.byref(m),
                                            dptr(signals.contiguous()), C.byref(g), C.byref(mk),
                                            C.byref(c), reps.ctypes.data_as(C.POINTER(C.c_double)),
                                            dptr(img), dptr(sos),
                                            th.ctypes.data_as(C.POINTER(C.c_double))))
    return reps, img, sos, th


def joint_reconstruct_batch(ctx: Context, signals: list, ring: RingGeometry, meta: SignalMetaInfo,
                            grid: GridSpec, mask: CircularMask, cfgs: list,
                            images: list | None = None, sos: list | None = None):
    """pact_joint_reconstruct_batch: joint_reconstruct of several frames of one
    geometry run concurrently (one engine stream each); identical results to
    separate joint_reconstruct calls.  `signals`, `images` and `sos` may be CUDA or
    host tensors (pinned host memory keeps the library's per-frame copies
    asynchronous; synchronise before reading host outputs).
    -> (reports [n, epochs, 4], images, sos, thetas)."""
    n = len(signals)
    assert len(cfgs) == n and n > 0
    cs = [c.c() for c in cfgs]  # keep each delays array alive
    carr = (_abi.TrainConfig * n)(*[c for c, _ in cs])
    # CUDA tensors, or host tensors (pinned: asynchronous) staged by the library
    sigs = [s.contiguous() for s in signals]
    for s in sigs:
        assert s.dtype == torch.float32 and s.numel() == ring.n_transducers * meta.n_samples, \
            "signals: fp32 [N, T] expected"
    for t in (images or []) + (sos or []):
        assert t.dtype == torch.float32 and t.is_contiguous() and \
            t.numel() == grid.width * grid.height, "images / sos: contiguous fp32 [H, W] expected"
    sig_p = (C.c_void_p * n)(*[s.data_ptr() for s in sigs])
    if images is None:
        images = [torch.empty((grid.height, grid.width), device="cuda", dtype=torch.float32)
                  for _ in range(n)]
    if sos is None:
        sos = [torch.empty((grid.height, grid.width), device="cuda", dtype=torch.float32)
               for _ in range(n)]
    img_p = (C.c_void_p * n)(*[t.data_ptr() for t in images])
    sos_p = (C.c_void_p * n)(*[t.data_ptr() for t in sos])
    c0 = cfgs[0]
    P = SirenSpec(c0.hidden, c0.sine_layers, c0.omega0, c0.out_scale,
                  meta.background_sos).param_count()
    reps = np.zeros((n, c0.epochs, 4))
    ths = np.zeros((n, P), np.float64)
    r, m, g, mk = ring.c(), meta.c(), grid.c(), mask.c()
    check(_abi.lib().pact_joint_reconstruct_batch(
        ctx.handle, n, C.byref(r), C.byref(m), sig_p, C.byref(g), C.byref(mk), carr,
        reps.ctypes.data_as(C.POINTER(C.c_double)), img_p, sos_p,
        ths.ctypes.data_as(C.POINTER(C.c_double))))
    return reps, images, sos, ths
