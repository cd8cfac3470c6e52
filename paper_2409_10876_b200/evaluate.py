"""Evaluation harness of the reference (proj/include/pact/evaluate.hpp), SURVEY §8(f)-4.

The metrics are GPU reductions in the library (`pact_psnr`, `pact_ssim`,
`pact_sos_rmse_masked`, csrc/metrics.cu); `benchmark` composes the four
reconstruction methods of evaluate.hpp:164-220 from the library's entry points
(das, dual_sos_das, deconvolve_image with the true SOS, joint_reconstruct) and
scores them against the unaberrated DAS reference (evaluate.hpp:149-160).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from .api import (BodyModel, CircularMask, Context, DeconvolveOptions, GridSpec, RingGeometry,
                  SignalMetaInfo, TrainConfig, check, dptr, joint_reconstruct, make_patch_layout)


def _f64(x, shape=None) -> torch.Tensor:
    t = torch.as_tensor(x)
    t = t.to(device="cuda", dtype=torch.float64).contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError("raster shape mismatch")
    return t


def _same_shape(a: torch.Tensor, b: torch.Tensor, what: str):
    if tuple(a.shape) != tuple(b.shape):
        raise _abi.ValidationError(_abi.PACT_E_VALIDATION, f"{what}: image shapes differ")


def psnr(ctx: Context, test, truth, data_range: float) -> float:
    """psnr, evaluate.hpp:39-51 (+inf for identical images)."""
    a, b = _f64(test), _f64(truth)
    _same_shape(a, b, "psnr")
    out = C.c_double(0.0)
    check(_abi.lib().pact_psnr(ctx.handle, dptr(a), dptr(b), a.shape[1], a.shape[0],
                               float(data_range), C.byref(out)))
    return out.value


def ssim(ctx: Context, test, truth, data_range: float) -> float:
    """ssim, evaluate.hpp:53-96."""
    a, b = _f64(test), _f64(truth)
    _same_shape(a, b, "ssim")
    out = C.c_double(0.0)
    check(_abi.lib().pact_ssim(ctx.handle, dptr(a), dptr(b), a.shape[1], a.shape[0],
                               float(data_range), C.byref(out)))
    return out.value


def sos_rmse_masked(ctx: Context, test, truth, grid: GridSpec, mask: CircularMask) -> float:
    """sos_rmse_masked, evaluate.hpp:99-114."""
    a, b = _f64(test), _f64(truth)
    if tuple(a.shape) != tuple(b.shape):
        raise _abi.ValidationError(_abi.PACT_E_VALIDATION, "sos_rmse: shapes differ")
    out = C.c_double(0.0)
    g, m = grid.c(), mask.c()
    check(_abi.lib().pact_sos_rmse_masked(ctx.handle, dptr(a), dptr(b), C.byref(g), C.byref(m),
                                          C.byref(out)))
    return out.value


# --------------------------------------------------------------------------- #
# benchmark (evaluate.hpp:117-220)
# --------------------------------------------------------------------------- #

@dataclass
class Phantom:
    """Phantom, phantom.hpp:76-84: pressure and SOS rasters on `grid`, the TOF mask."""
    grid: GridSpec
    pressure: np.ndarray  # fp64 [H, W]
    sos: np.ndarray       # fp64 [H, W], m/s
    mask: CircularMask
    background_sos: float


@dataclass
class EvalReport:
    method: str
    psnr: float = 0.0
    ssim: float = 0.0
    sos_rmse: float = 0.0  # m/s over the mask
    runtime: float = 0.0   # s


@dataclass
class BenchmarkEntry:
    report: EvalReport
    image: torch.Tensor
    sos: np.ndarray


@dataclass
class BenchmarkConfig:
    """BenchmarkConfig, evaluate.hpp:132-140."""
    grid: GridSpec
    das_v0: float = 1510.0
    das_delay: float = 0.0
    body: BodyModel = field(default_factory=lambda: BodyModel(0.0, 0.0, 9.0, 1561.0))
    train: TrainConfig = field(default_factory=TrainConfig)
    pulse_sigma: float = 100e-9  # SimulateOptions of the unaberrated reference
    ray_step: float = 0.05


METHODS = ("das", "dual_sos", "deconv_true_sos", "nf_apact")


def normalize_for_metrics(img: torch.Tensor, ref_max: float) -> torch.Tensor:
    """normalize_for_metrics, evaluate.hpp:143-147."""
    return (img.double() / ref_max).clamp(0.0, 1.0)


def unaberrated_reference(ctx: Context, truth: Phantom, ring: RingGeometry, meta: SignalMetaInfo,
                          grid: GridSpec, cfg: BenchmarkConfig) -> torch.Tensor:
    """unaberrated_reference, evaluate.hpp:149-160: the same phantom simulated with
    SOS = v0 everywhere, reconstructed by DAS at d = 0."""
    uniform = np.full_like(truth.sos, truth.background_sos)
    sig = ctx.simulate_signals(truth.grid, truth.pressure, uniform, truth.mask,
                               truth.background_sos, ring, meta, cfg.pulse_sigma, cfg.ray_step)
    return ctx.das(sig, ring, meta, grid, truth.background_sos, 0.0)


def _sos_raster_constant(truth: Phantom, v: float) -> np.ndarray:
    return np.full_like(truth.sos, v)


def benchmark(ctx: Context, signals: torch.Tensor, ring: RingGeometry, meta: SignalMetaInfo,
              truth: Phantom, methods, cfg: BenchmarkConfig) -> list[BenchmarkEntry]:
    """benchmark, evaluate.hpp:164-220 (methods run sequentially; runtime is wall clock
    around each method, device work included)."""
    for m in methods:
        if m not in METHODS:
            raise _abi.ValidationError(_abi.PACT_E_VALIDATION, f"benchmark: unknown method '{m}'")
    v0 = meta.background_sos
    ref = unaberrated_reference(ctx, truth, ring, meta, cfg.grid, cfg)
    ref_max = float(ref.abs().max().item())
    if not ref_max > 0.0:
        raise _abi.ValidationError(_abi.PACT_E_VALIDATION, "benchmark: empty reference image")
    ref_norm = normalize_for_metrics(ref, ref_max)
    out = []
    for m in methods:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if m == "das":
            image = ctx.das(signals, ring, meta, cfg.grid, cfg.das_v0, cfg.das_delay)
            sos = _sos_raster_constant(truth, cfg.das_v0)
        elif m == "dual_sos":
            image = ctx.dual_sos_das(signals, ring, meta, cfg.grid, v0, cfg.body)
            sos = _sos_raster_constant(truth, v0)
            g = truth.grid
            xs = g.origin_x + np.arange(g.width) * g.pitch
            ys = g.origin_y + np.arange(g.height) * g.pitch
            X, Y = np.meshgrid(xs, ys)
            inside = np.hypot(X - cfg.body.center_x, Y - cfg.body.center_y) <= cfg.body.radius
            sos[inside] = cfg.body.body_sos
        elif m == "deconv_true_sos":
            tc = cfg.train
            stack = ctx.das_stack(signals, ring, meta, cfg.grid, v0, tc.delays)
            layout = make_patch_layout(cfg.grid, tc.patch_mm, tc.overlap)
            sos_dev = torch.as_tensor((truth.sos - v0).astype(np.float32)).cuda()
            image = ctx.deconvolve_image(stack, tc.delays, v0, sos_dev, ring, truth.mask, layout,
                                         DeconvolveOptions(tc.eps_deconv, tc.n_angles, tc.ray_step,
                                                           tc.merge_fwhm))
            sos = truth.sos
        else:  # nf_apact
            _, image, sos_t, _ = joint_reconstruct(ctx, signals, ring, meta, cfg.grid, truth.mask,
                                                   cfg.train)
            sos = sos_t.double().cpu().numpy()
        torch.cuda.synchronize()
        rep = EvalReport(m, runtime=time.perf_counter() - t0)
        test_norm = normalize_for_metrics(image, ref_max)
        rep.psnr = psnr(ctx, test_norm, ref_norm, 1.0)
        rep.ssim = ssim(ctx, test_norm, ref_norm, 1.0)
        rep.sos_rmse = sos_rmse_masked(ctx, sos, truth.sos, truth.grid, truth.mask)
        out.append(BenchmarkEntry(rep, image, sos))
    return out
