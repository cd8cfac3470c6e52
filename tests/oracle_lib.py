"""TEST INFRASTRUCTURE: ctypes view of the CPU oracle builds.

orc = oracle/liboracle.so (the C restatement, oracle/pact_oracle.c)
ref = oracle/_ref/libpact_ref.so (the reference headers compiled in place;
      absent on a GPU box unless the prebuilt file travelled with the repo).
Both export the same signatures with prefixes orc_ / ref_ (a function the
restatement does not provide is simply missing from orc).
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


class TrainCfg(C.Structure):
    """RefTrainCfg of oracle/ref_shim.cpp (TrainConfig, optimize.hpp:48-69)."""
    _fields_ = [("epochs", C.c_int), ("steps_per_epoch", C.c_int), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("adam_eps", C.c_double),
                ("lambda_tv", C.c_double), ("n_delays", C.c_int),
                ("delays", C.POINTER(C.c_double)), ("eps_deconv", C.c_double),
                ("n_angles", C.c_int), ("ray_step", C.c_double), ("seed", C.c_uint64),
                ("hidden", C.c_int), ("sine_layers", C.c_int), ("omega0", C.c_double),
                ("out_scale", C.c_double), ("patch_mm", C.c_double), ("overlap", C.c_double),
                ("merge_fwhm", C.c_double), ("implicit_xhat_grad", C.c_int), ("workers", C.c_int)]


def train_cfg(cfg) -> tuple[TrainCfg, object]:
    """From paper_2409_10876_b200.api.TrainConfig (or any object with its fields)."""
    arr = (C.c_double * len(cfg.delays))(*[float(d) for d in cfg.delays])
    c = TrainCfg(cfg.epochs, cfg.steps_per_epoch, cfg.learning_rate, cfg.beta1, cfg.beta2,
                 cfg.adam_eps, cfg.lambda_tv, len(cfg.delays), C.cast(arr, C.POINTER(C.c_double)),
                 cfg.eps_deconv, cfg.n_angles, cfg.ray_step, cfg.seed, cfg.hidden,
                 cfg.sine_layers, cfg.omega0, cfg.out_scale, cfg.patch_mm, cfg.overlap,
                 cfg.merge_fwhm, 1 if cfg.implicit_xhat_grad else 0, cfg.workers)
    return c, arr


SIGS = {
    "das_stack": [_I, _D, _D, _I, _D, _D, _P, _I, _I, _D, _D, _D, _D, _I, _P, _I, _P],
    "dual_sos_das": [_I, _D, _D, _I, _D, _D, _P, _I, _I, _D, _D, _D, _D, _D, _D, _D, _D, _P],
    "psnr": [_P, _P, _I, _I, _D, _P],
    "ssim": [_P, _P, _I, _I, _D, _P],
    "sos_rmse_masked": [_P, _P, _I, _I, _D, _D, _D, _D, _D, _D, _P],
    "init_siren": [C.c_uint64, _I, _I, _D, _D, _D, _P],
    "render_sos": [_I, _I, _D, _D, _D, _P, _I, _I, _D, _D, _D, _D, _D, _D, _P, _P],
    "backprop_sos": [_I, _I, _D, _D, _D, _P, _I, _I, _D, _D, _D, _D, _D, _D, _P, _P],
    "wavefront_profile": [_I, _P, _I, _D, _D, _I, _I, _D, _D, _D, _P, _D, _D, _D, _D, _I, _D, _P],
    "transfer_stack": [_I, _P, _I, _P, _I, _D, _P],
    "patch_layout": [_I, _I, _D, _D, _D, _D, _D, _P, _P, _P],
    "patch_spectra": [_I, _P, _D, _I, _I, _D, _D, _D, _P, _D, _D, _I, _P],
    "deconvolve_image": [_I, _P, _D, _I, _I, _D, _D, _D, _P, _P, _I, _D, _D, _D, _D, _D, _D, _D,
                         _D, _I, _D, _D, _I, _P],
    "fused_patch_loss_grad": [_I, _P, _P, _I, _D, _I, _P, _D, _D, _I, _P, _P],
    "wavefront_grad_trace": [_D, _D, _I, _D, _D, _I, _I, _D, _D, _D, _P, _D, _D, _D, _D, _I, _D,
                             _P, _P],
    "tv_loss": [_I, _I, _D, _D, _D, _P, _D, _D, _D, _D, _P, _P],
    "adam_step": [_I, _P, _P, _P, _P, _P, _D, _D, _D, _D],
    "joint_reconstruct": [_I, _D, _D, _I, _D, _D, _D, _P, _I, _I, _D, _D, _D, _D, _D, _D,
                          C.POINTER(TrainCfg), _P, _P, _P, _P],
    "nf_step": [_I, _D, _D, _I, _D, _D, _D, _P, _I, _I, _D, _D, _D, _D, _D, _D,
                C.POINTER(TrainCfg), _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "small_instance_signals": [_P, _P, _P],
    "simulate_signals": [_I, _I, _D, _D, _D, _P, _P, _D, _D, _D, _D, _I, _D, _D, _D, _D, _D, _I,
                         _D, _I, _P],
}


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _g(grid):
    return (grid.width, grid.height, grid.pitch, grid.origin_x, grid.origin_y)


def _r(ring):
    return (ring.n_transducers, ring.radius, ring.angle_offset)


def _m(mask):
    return (mask.center_x, mask.center_y, mask.radius)


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

    def has(self, name) -> bool:
        return hasattr(self.lib, self.prefix + name)

    def call(self, name, *args):
        rc = getattr(self.lib, self.prefix + name)(*args)
        if rc != 0:
            raise RuntimeError(f"{self.prefix}{name} failed with code {rc}")

    # -- part 1 -----------------------------------------------------------
    def das_stack(self, sig, ring, meta, grid, v0, delays, workers=0):
        sig = _f64(sig)
        d = _f64(delays)
        out = np.zeros((len(d), grid.height, grid.width))
        self.call("das_stack", *_r(ring), meta.n_samples, meta.dt, meta.t0, _p(sig), *_g(grid),
                  v0, len(d), _p(d), workers, _p(out))
        return out

    def dual_sos_das(self, sig, ring, meta, grid, v0, body):
        sig = _f64(sig)
        out = np.zeros((grid.height, grid.width))
        self.call("dual_sos_das", *_r(ring), meta.n_samples, meta.dt, meta.t0, _p(sig), *_g(grid),
                  v0, body.center_x, body.center_y, body.radius, body.body_sos, _p(out))
        return out

    # -- metrics (evaluate.hpp:39-114) -------------------------------------
    def psnr(self, test, truth, data_range):
        a, b = _f64(test), _f64(truth)
        out = np.zeros(1)
        self.call("psnr", _p(a), _p(b), a.shape[1], a.shape[0], data_range, _p(out))
        return float(out[0])

    def ssim(self, test, truth, data_range):
        a, b = _f64(test), _f64(truth)
        out = np.zeros(1)
        self.call("ssim", _p(a), _p(b), a.shape[1], a.shape[0], data_range, _p(out))
        return float(out[0])

    def sos_rmse_masked(self, test, truth, grid, mask):
        a, b = _f64(test), _f64(truth)
        out = np.zeros(1)
        self.call("sos_rmse_masked", _p(a), _p(b), *_g(grid), *_m(mask), _p(out))
        return float(out[0])

    # -- SIREN ------------------------------------------------------------
    def init_siren(self, seed, spec, n_params):
        th = np.zeros(n_params)
        self.call("init_siren", seed, spec.hidden, spec.n_hidden_layers, spec.omega0,
                  spec.out_scale, spec.v0, _p(th))
        return th

    def render_sos(self, spec, theta, grid, mask):
        th = _f64(theta)
        out = np.zeros((grid.height, grid.width))
        n = C.c_int(0)
        self.call("render_sos", spec.hidden, spec.n_hidden_layers, spec.omega0, spec.out_scale,
                  spec.v0, _p(th), *_g(grid), *_m(mask), _p(out), C.byref(n))
        return out

    def backprop_sos(self, spec, theta, grid, mask, grad_masked):
        th = _f64(theta)
        g = _f64(grad_masked)
        out = np.zeros(len(th))
        self.call("backprop_sos", spec.hidden, spec.n_hidden_layers, spec.omega0, spec.out_scale,
                  spec.v0, _p(th), *_g(grid), *_m(mask), _p(g), _p(out))
        return out

    # -- part 2 -----------------------------------------------------------
    def wavefront_profile(self, centers, ring, grid, sos, v0, mask, n_angles, step):
        cen = _f64(centers).reshape(-1, 2)
        s = _f64(sos)
        w = np.zeros((cen.shape[0], n_angles))
        self.call("wavefront_profile", cen.shape[0], _p(cen), *_r(ring), *_g(grid), _p(s), v0,
                  *_m(mask), n_angles, step, _p(w))
        return w

    def transfer_stack(self, w, delays, P, pitch):
        w = _f64(w)
        d = _f64(delays)
        H = np.zeros((len(d), P, P), np.complex128)
        self.call("transfer_stack", len(w), _p(w), len(d), _p(d), P, pitch, _p(H))
        return H

    def patch_layout(self, grid, patch_mm, overlap):
        info = np.zeros(4, np.int32)
        self.call("patch_layout", *_g(grid), patch_mm, overlap, _p(info), None, None)
        n = int(info[2] * info[3])
        off = np.zeros((n, 2), np.int32)
        cen = np.zeros((n, 2))
        self.call("patch_layout", *_g(grid), patch_mm, overlap, _p(info), _p(off), _p(cen))
        return dict(P=int(info[0]), stride=int(info[1]), nx=int(info[2]), ny=int(info[3]),
                    offsets=off, centers=cen)

    def patch_spectra(self, stack, delays, v0, grid, patch_mm, overlap, workers=0):
        st = _f64(stack)
        d = _f64(delays)
        lay = self.patch_layout(grid, patch_mm, overlap)
        P = lay["P"]
        Y = np.zeros((len(lay["offsets"]), len(d), P, P), np.complex128)
        self.call("patch_spectra", len(d), _p(d), v0, *_g(grid), _p(st), patch_mm, overlap,
                  workers, _p(Y))
        return Y

    def deconvolve_image(self, stack, delays, v0, grid, sos, ring, mask, patch_mm, overlap, eps,
                         n_angles, ray_step, merge_fwhm, workers=0):
        st = _f64(stack)
        d = _f64(delays)
        s = _f64(sos)
        img = np.zeros((grid.height, grid.width))
        self.call("deconvolve_image", len(d), _p(d), v0, *_g(grid), _p(st), _p(s), *_r(ring),
                  *_m(mask), patch_mm, overlap, eps, n_angles, ray_step, merge_fwhm, workers,
                  _p(img))
        return img

    # -- part 3 -----------------------------------------------------------
    def fused_patch_loss_grad(self, Y, w, P, pitch, n_angles, delays, eps, scale, implicit=True):
        Yf = np.ascontiguousarray(np.asarray(Y, np.complex64))
        ww = _f64(w)
        d = _f64(delays)
        loss = C.c_double(0)
        dw = np.zeros(n_angles)
        self.call("fused_patch_loss_grad", len(d), _p(Yf), _p(ww), P, pitch, n_angles, _p(d), eps,
                  scale, 1 if implicit else 0, C.byref(loss), _p(dw))
        return loss.value, dw

    def wavefront_grad_trace(self, center, ring, grid, sos, v0, mask, n_angles, step, dw,
                             grad_v=None):
        s = _f64(sos)
        g = np.zeros((grid.height, grid.width)) if grid_v_is_none(grad_v) else _f64(grad_v).copy()
        d = _f64(dw)
        self.call("wavefront_grad_trace", float(center[0]), float(center[1]), *_r(ring), *_g(grid),
                  _p(s), v0, *_m(mask), n_angles, step, _p(d), _p(g))
        return g

    def tv_loss(self, grid, raster, mask, lam):
        r = _f64(raster)
        n = int(np.count_nonzero(_mask_flags(grid, mask)))
        g = np.zeros(max(n, 1))
        val = C.c_double(0)
        self.call("tv_loss", *_g(grid), _p(r), *_m(mask), lam, C.byref(val), _p(g))
        return val.value, g[:n]

    def adam_step(self, params, grads, m, v, t, lr, b1, b2, eps):
        p = _f64(params).copy()
        g = _f64(grads)
        mm = _f64(m).copy()
        vv = _f64(v).copy()
        tt = C.c_long(t)
        self.call("adam_step", len(p), _p(p), _p(g), _p(mm), _p(vv), C.byref(tt), lr, b1, b2, eps)
        return p, mm, vv, tt.value

    # -- engine -----------------------------------------------------------
    def nf_step(self, sig, ring, meta, grid, mask, cfg, theta, patch_lo=0, patch_hi=-1,
                want_image=True):
        c, arr = train_cfg(cfg)
        sig = _f64(sig)
        th = _f64(theta)
        lay = self.patch_layout(grid, cfg.patch_mm, cfg.overlap)
        n = len(lay["offsets"])
        nm = int(np.count_nonzero(_mask_flags(grid, mask)))
        data = C.c_double(0)
        tv = C.c_double(0)
        secs = C.c_double(0)
        out = dict(loss_patch=np.zeros(n), w=np.zeros((n, cfg.n_angles)),
                   dw=np.zeros((n, cfg.n_angles)), sos=np.zeros((grid.height, grid.width)),
                   grad_v_masked=np.zeros(max(nm, 1)), grad_theta=np.zeros(len(th)),
                   image=np.zeros((grid.height, grid.width)) if want_image else None)
        self.call("nf_step", *_r(ring), meta.n_samples, meta.dt, meta.t0, meta.background_sos,
                  _p(sig), *_g(grid), *_m(mask), C.byref(c), _p(th), patch_lo, patch_hi,
                  C.byref(data), C.byref(tv), _p(out["loss_patch"]), _p(out["w"]), _p(out["dw"]),
                  _p(out["sos"]), _p(out["grad_v_masked"]), _p(out["grad_theta"]),
                  _p(out["image"]), C.byref(secs))
        out.update(data_term=data.value, tv_term=tv.value, seconds=secs.value)
        out["grad_v_masked"] = out["grad_v_masked"][:nm]
        return out

    # -- composed (non-fused) path, one patch per call (ref_shim.cpp) -----
    def _fn(self, name, args, res=C.c_int):
        fn = getattr(self.lib, self.prefix + name)
        fn.argtypes = args
        fn.restype = res
        return fn

    def _ok(self, name, rc):
        if rc != 0:
            raise RuntimeError(f"{self.prefix}{name} failed ({rc}): {self.last_error()}")

    def multichannel_deconvolve(self, Y, H, eps):
        """Y, H complex128 [K, P, P] -> X complex128 [P, P]."""
        Y = np.ascontiguousarray(Y, np.complex128)
        H = np.ascontiguousarray(H, np.complex128)
        K, P = Y.shape[0], Y.shape[1]
        X = np.zeros((P, P), np.complex128)
        self._ok("multichannel_deconvolve", self._fn("multichannel_deconvolve",
                 [_I, _I, _P, _P, _D, _P])(K, P, _p(Y), _p(H), eps, _p(X)))
        return X

    def deconv_jacobian_H(self, Y, H, eps, j, b):
        Y = np.ascontiguousarray(Y, np.complex128)
        H = np.ascontiguousarray(H, np.complex128)
        out = np.zeros(4)
        self._ok("deconv_jacobian_H", self._fn("deconv_jacobian_H",
                 [_I, _I, _P, _P, _D, _I, _I, _P])(Y.shape[0], Y.shape[1], _p(Y), _p(H), eps, j, b,
                                                   _p(out)))
        return complex(out[0], out[1]), complex(out[2], out[3])

    def patch_data_loss(self, Y, H, pitch, eps, scale, implicit=True):
        Y = np.ascontiguousarray(Y, np.complex128)
        H = np.ascontiguousarray(H, np.complex128)
        loss = C.c_double()
        g = np.zeros_like(Y)
        self._ok("patch_data_loss", self._fn("patch_data_loss",
                 [_I, _I, _D, _P, _P, _D, _D, _I, _P, _P])(
                     Y.shape[0], Y.shape[1], pitch, _p(Y), _p(H), eps, scale, 1 if implicit else 0,
                     C.byref(loss), _p(g)))
        return loss.value, g

    def data_loss(self, Y, H, pitch, eps, implicit=True):
        """Y, H complex128 [n, K, P, P] -> (value, grad_h)."""
        Y = np.ascontiguousarray(Y, np.complex128)
        H = np.ascontiguousarray(H, np.complex128)
        val = C.c_double()
        g = np.zeros_like(Y)
        self._ok("data_loss", self._fn("data_loss", [_I, _I, _I, _D, _P, _P, _D, _I, _P, _P])(
            Y.shape[0], Y.shape[1], Y.shape[2], pitch, _p(Y), _p(H), eps, 1 if implicit else 0,
            C.byref(val), _p(g)))
        return val.value, g

    def transfer_grad_to_wavefront(self, w, delays, P, pitch, grad_h):
        w = _f64(w)
        d = _f64(delays)
        g = np.ascontiguousarray(grad_h, np.complex128)
        dw = np.zeros(len(w))
        self._ok("transfer_grad_to_wavefront", self._fn("transfer_grad_to_wavefront",
                 [_I, _P, _I, _P, _I, _D, _P, _P])(len(w), _p(w), len(d), _p(d), P, pitch, _p(g),
                                                   _p(dw)))
        return dw

    def wavefront_jacobian(self, center, ring, grid, sos, v0, mask, n_angles, step, dw=None,
                           grad_v=None):
        """-> (w [A], counts [A], pixel, dw_dv[, grad_v after J^T dw])."""
        s = _f64(sos)
        fn = self._fn("wavefront_jacobian", [_D, _D, _I, _D, _D, _I, _I, _D, _D, _D, _P, _D, _D, _D,
                                             _D, _I, _D, _P, _P, _P, _P, C.c_long, _P, _P])
        w = np.zeros(n_angles)
        counts = np.zeros(n_angles, np.int64)
        args = (float(center[0]), float(center[1]), *_r(ring), *_g(grid), _p(s), v0, *_m(mask),
                n_angles, step)
        self._ok("wavefront_jacobian", fn(*args, _p(w), _p(counts), None, None, 0, None, None))
        nnz = int(counts.sum())
        pix = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1), np.float32)
        gv = None
        if dw is not None:
            gv = np.zeros((grid.height, grid.width)) if grad_v is None else _f64(grad_v).copy()
        self._ok("wavefront_jacobian", fn(*args, _p(w), _p(counts), _p(pix), _p(val), nnz,
                                          None if dw is None else _p(_f64(dw)), _p(gv)))
        return w, counts, pix[:nnz], val[:nnz], gv

    def merge_patches(self, grid, patch_mm, overlap, patches, fwhm):
        ps = _f64(patches)
        img = np.zeros((grid.height, grid.width))
        self._ok("merge_patches", self._fn("merge_patches", [_I, _I, _D, _D, _D, _D, _D, _P, _D, _P])(
            *_g(grid), patch_mm, overlap, _p(ps), fwhm, _p(img)))
        return img

    # -- CPU-baseline session (ref_shim.cpp ref_nf_session_*) -----------
    def nf_session(self, sig, ring, meta, grid, mask, cfg):
        """joint_reconstruct's one-time setup (optimize.hpp:374-405), once;
        returns (handle, setup seconds).  Close with nf_session_close."""
        c, arr = train_cfg(cfg)
        sig = _f64(sig)
        secs = C.c_double(0)
        fn = self.lib.ref_nf_session_open
        fn.restype = C.c_void_p
        fn.argtypes = [_I, _D, _D, _I, _D, _D, _D, _P, _I, _I, _D, _D, _D, _D, _D, _D,
                       C.POINTER(TrainCfg), _P]
        h = fn(*_r(ring), meta.n_samples, meta.dt, meta.t0, meta.background_sos, _p(sig),
               *_g(grid), *_m(mask), C.byref(c), C.byref(secs))
        if not h:
            raise RuntimeError("ref_nf_session_open failed: " + self.last_error())
        return h, secs.value

    def nf_session_step(self, h, workers, patch_lo=0, patch_hi=-1, with_siren=True):
        """One step of optimize.hpp:413-467 -> dict of phase seconds + data term."""
        t = np.zeros(6)
        data = C.c_double(0)
        fn = self.lib.ref_nf_session_step
        fn.argtypes = [_P, _I, _I, _I, _I, _P, _P]
        fn.restype = C.c_int
        rc = fn(C.c_void_p(h), workers, patch_lo, patch_hi, 1 if with_siren else 0, _p(t),
                C.byref(data))
        if rc != 0:
            raise RuntimeError("ref_nf_session_step failed: " + self.last_error())
        keys = ("render", "patches", "tv", "backprop", "adam", "total")
        out = dict(zip(keys, t.tolist()))
        out["data_term"] = data.value
        return out

    def nf_session_close(self, h):
        fn = self.lib.ref_nf_session_close
        fn.argtypes = [_P]
        fn.restype = None
        fn(C.c_void_p(h))

    def last_error(self) -> str:
        fn = getattr(self.lib, self.prefix + "last_error", None)
        if fn is None:
            return ""
        fn.restype = C.c_char_p
        return (fn() or b"").decode()

    def param_count(self, hidden, layers) -> int:
        fn = self.lib.ref_siren_param_count
        fn.argtypes = [_I, _I]
        fn.restype = C.c_long
        return int(fn(hidden, layers))

    def simulate(self, w, pressure, sos, sim_mask, workers=0, ring=None):
        """simulate_signals (phantom.hpp:282-362) of rasters on w.grid, with
        the caller's window (w.meta) -> fp64 [N, T]."""
        g = w.grid
        ring = ring or w.ring
        out = np.zeros((ring.n_transducers, w.meta.n_samples))
        pr, so = _f64(pressure), _f64(sos)
        self.call("simulate_signals", g.width, g.height, g.pitch, g.origin_x, g.origin_y, _p(pr),
                  _p(so), *_m(sim_mask), w.v0, *_r(ring), 100e-9, w.meta.dt, w.meta.t0,
                  w.meta.n_samples, w.ray_step, workers, _p(out))
        return out

    def joint_reconstruct(self, sig, ring, meta, grid, mask, cfg, n_params):
        c, arr = train_cfg(cfg)
        sig = _f64(sig)
        reports = np.zeros((cfg.epochs, 4))
        img = np.zeros((grid.height, grid.width))
        sos = np.zeros((grid.height, grid.width))
        th = np.zeros(n_params)
        self.call("joint_reconstruct", *_r(ring), meta.n_samples, meta.dt, meta.t0,
                  meta.background_sos, _p(sig), *_g(grid), *_m(mask), C.byref(c), _p(reports),
                  _p(img), _p(sos), _p(th))
        return reports, img, sos, th


def grid_v_is_none(x):
    return x is None


def _mask_flags(grid, mask):
    xs = grid.origin_x + np.arange(grid.width) * grid.pitch
    ys = grid.origin_y + np.arange(grid.height) * grid.pitch
    X, Y = np.meshgrid(xs, ys)
    return np.hypot(X - mask.center_x, Y - mask.center_y) <= mask.radius


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
    a = np.asarray(a)
    b = np.asarray(b)
    dt = np.complex128 if (np.iscomplexobj(a) or np.iscomplexobj(b)) else np.float64
    a = a.astype(dt)
    b = b.astype(dt)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den > 0 else 1.0))
