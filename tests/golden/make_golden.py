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


def dual_case(R):
    """dual_sos_das (beamform.hpp:124-150): a body disc overlapping part of a
    small grid, a window that clips some taps, i.i.d. signals."""
    from paper_2409_10876_b200.api import BodyModel

    rng = np.random.default_rng(4321)
    ring = RingGeometry(48, 30.0, 0.05)
    meta = SignalMetaInfo(600, 25e-9, 14.0e-6, 1500.0)
    grid = GridSpec(40, 36, 0.3, -5.85, -5.25)
    sig = rng.standard_normal((48, 600)).astype(np.float32).astype(np.float64)
    bodies = [BodyModel(1.0, -0.5, 5.0, 1580.0), BodyModel(-2.0, 1.5, 9.0, 1420.0)]
    outs = [R.dual_sos_das(sig, ring, meta, grid, 1500.0, b) for b in bodies]
    save("dual_das", ring=ring_arr(ring), meta=meta_arr(meta), grid=grid_arr(grid),
         sig=sig.astype(np.float32), v0=np.array(1500.0),
         bodies=np.array([[b.center_x, b.center_y, b.radius, b.body_sos] for b in bodies]),
         out=np.stack(outs))


def metrics_case(R):
    """psnr / ssim / sos_rmse_masked (evaluate.hpp:39-114) on random and
    structured images (a blob field and its 5-pixel shift, test_evaluate.cpp:83-104)."""
    from paper_2409_10876_b200.api import CircularMask

    rng = np.random.default_rng(777)
    a = rng.uniform(0, 1, (36, 40))
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
    yy, xx = np.mgrid[0:64, 0:64]
    img = sum(amp * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / 18.0)
              for cx, cy, amp in [(20, 22, 1.0), (40, 35, 0.8), (30, 48, 0.6)])
    shifted = np.zeros_like(img)
    shifted[:, 5:] = img[:, :-5]
    grid = GridSpec(33, 29, 0.1, -1.6, -1.4)
    sos_t = 1500 + 40 * rng.uniform(0, 1, (29, 33))
    sos_r = 1500 + 40 * rng.uniform(0, 1, (29, 33))
    mask = CircularMask(0.2, -0.1, 1.2)
    vals = np.array([R.psnr(b, a, 1.0), R.ssim(b, a, 1.0), R.psnr(shifted, img, 1.0),
                     R.ssim(shifted, img, 1.0), R.sos_rmse_masked(sos_r, sos_t, grid, mask)])
    save("metrics", a=a, b=b, img=img, shifted=shifted, grid=grid_arr(grid), sos_t=sos_t,
         sos_r=sos_r, mask=np.array([mask.center_x, mask.center_y, mask.radius]), vals=vals)


def small_case(R):
    """testsupport::SmallInstance (proj/tests/test_support.hpp:38-75), through
    every hot-path entry point of the reference."""
    import ctypes as C

    import golden_util as gu
    from paper_2409_10876_b200.api import SirenSpec

    si = gu.small_instance()
    T = C.c_int(0)
    t0 = C.c_double(0)
    R.call("small_instance_signals", None, C.byref(T), C.byref(t0))
    sig = np.zeros((si.ring.n_transducers, T.value))
    R.call("small_instance_signals", sig.ctypes.data_as(C.c_void_p), C.byref(T), C.byref(t0))
    sig = sig.astype(np.float32).astype(np.float64)  # both sides consume fp32 values
    meta = SignalMetaInfo(T.value, 25e-9, t0.value, 1500.0)
    cfg = si.cfg
    spec = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, 1500.0)
    n_params = spec.param_count()
    theta0 = R.init_siren(0, spec, n_params)
    theta2 = R.init_siren(2, spec, n_params)
    stack = R.das_stack(sig, si.ring, meta, si.grid, 1500.0, cfg.delays, workers=1)
    Y = R.patch_spectra(stack, cfg.delays, 1500.0, si.grid, cfg.patch_mm, cfg.overlap, 1)
    step = R.nf_step(sig, si.ring, meta, si.grid, si.mask, cfg, theta2)
    lay = R.patch_layout(si.grid, cfg.patch_mm, cfg.overlap)
    H0 = R.transfer_stack(step["w"][0], cfg.delays, lay["P"], si.grid.pitch)
    tv_val, tv_grad = R.tv_loss(si.grid, step["sos"], si.mask, cfg.lambda_tv)
    from dataclasses import replace

    jcfg = replace(cfg, epochs=3, steps_per_epoch=2, seed=5)
    reports, jimg, jsos, jtheta = R.joint_reconstruct(sig, si.ring, meta, si.grid, si.mask, jcfg,
                                                      n_params)
    # deconvolve_image under the rendered SOS (deconv.hpp:176-198)
    dimg = R.deconvolve_image(stack, cfg.delays, 1500.0, si.grid, step["sos"], si.ring, si.mask,
                              cfg.patch_mm, cfg.overlap, cfg.eps_deconv, cfg.n_angles,
                              cfg.ray_step, cfg.merge_fwhm, 1)
    save("small_instance", sig=sig.astype(np.float32), meta=meta_arr(meta), theta0=theta0,
         theta2=theta2, stack=stack, Y=Y.astype(np.complex64), sos=step["sos"], w=step["w"],
         dw=step["dw"], loss_patch=step["loss_patch"], data_term=np.array(step["data_term"]),
         tv_term=np.array(step["tv_term"]), grad_v_masked=step["grad_v_masked"],
         grad_theta=step["grad_theta"], image=step["image"], H0=H0, tv_value=np.array(tv_val),
         tv_grad=tv_grad, deconv=dimg, reports=reports, joint_image=jimg, joint_sos=jsos,
         joint_theta=jtheta)


def cfg2_case(R):
    """BASELINE configs[1] (cfg2, Appendix A): simulated signals, one forward +
    gradient evaluation at the seed-0 SIREN, and the deconvolved image."""
    from paper_2409_10876_b200.api import CircularMask, SirenSpec

    w = wl.cfg2()
    sig = gu_simulate(R, w, seed=0)
    cfg = wl.train_config(w)
    spec = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, w.v0)
    theta = R.init_siren(0, spec, spec.param_count())
    step = R.nf_step(sig, w.ring, w.meta, w.grid, w.mask, cfg, theta)
    g = w.grid
    crop = GridSpec(32, 32, g.pitch, g.origin_x + 100 * g.pitch, g.origin_y + 60 * g.pitch)
    das_crop = R.das_stack(sig, w.ring, w.meta, crop, w.v0, cfg.delays)
    lay = R.patch_layout(g, cfg.patch_mm, cfg.overlap)
    H24 = R.transfer_stack(step["w"][24], cfg.delays, lay["P"], g.pitch)
    save("cfg2_step", sig=sig.astype(np.float32), theta=theta, das_crop=das_crop.astype(np.float32),
         crop=grid_arr(crop), sos=step["sos"].astype(np.float32), w=step["w"], dw=step["dw"],
         loss_patch=step["loss_patch"], data_term=np.array(step["data_term"]),
         tv_term=np.array(step["tv_term"]), grad_theta=step["grad_theta"],
         image=step["image"].astype(np.float32), H24=H24.astype(np.complex64))


def cfg2_wide_case(R, hidden, name):
    """cfg2's geometry and signals (the cfg2_step fixture) with a wider network,
    SIREN 2 -> hidden x 4 -> 1 (128: cfg3's, 256: cfg5's): one forward +
    gradient evaluation through the reference, for the tcgen05 SIREN kernels
    inside the training step."""
    from dataclasses import replace

    from paper_2409_10876_b200.api import SirenSpec

    w = replace(wl.cfg2(), hidden=hidden, sine_layers=4)
    sig = np.load(os.path.join(HERE, "cfg2_step.npz"))["sig"].astype(np.float64)
    cfg = wl.train_config(w)
    spec = SirenSpec(cfg.hidden, cfg.sine_layers, cfg.omega0, cfg.out_scale, w.v0)
    theta = R.init_siren(0, spec, spec.param_count())
    step = R.nf_step(sig, w.ring, w.meta, w.grid, w.mask, cfg, theta, want_image=False)
    save(name, theta=theta, sos=step["sos"].astype(np.float32), w=step["w"],
         dw=step["dw"], data_term=np.array(step["data_term"]), tv_term=np.array(step["tv_term"]),
         grad_theta=step["grad_theta"])


def gu_simulate(R, w, seed):
    """simulate_signals (phantom.hpp:282-362) of the Appendix A phantom, through
    the reference; SOS mask = disc of the image half-diagonal (D5)."""
    import math

    p, sos = wl.phantom_rasters(w, seed)
    g = w.grid
    r_half = math.hypot((g.width - 1) * g.pitch / 2, (g.height - 1) * g.pitch / 2) + g.pitch
    out = np.zeros((w.ring.n_transducers, w.meta.n_samples))
    pr = np.ascontiguousarray(p)
    so = np.ascontiguousarray(sos)
    import ctypes as C

    R.call("simulate_signals", g.width, g.height, g.pitch, g.origin_x, g.origin_y,
           pr.ctypes.data_as(C.c_void_p), so.ctypes.data_as(C.c_void_p), 0.0, 0.0, r_half, w.v0,
           w.ring.n_transducers, w.ring.radius, w.ring.angle_offset, 100e-9, w.meta.dt, w.meta.t0,
           w.meta.n_samples, 0.05, 0, out.ctypes.data_as(C.c_void_p))
    return out.astype(np.float32).astype(np.float64)


def main():
    R = ref()
    if R is None:
        sys.exit("oracle/_ref/libpact_ref.so missing: make -C oracle ref")
    which = sys.argv[1:] or ["das", "dual", "metrics", "small", "cfg2", "cfg2_h128", "cfg2_h256"]
    if "das" in which:
        das_cases(R)
    if "dual" in which:
        dual_case(R)
    if "metrics" in which:
        metrics_case(R)
    if "small" in which:
        small_case(R)
    if "cfg2" in which:
        cfg2_case(R)
    if "cfg2_h128" in which:
        cfg2_wide_case(R, 128, "cfg2_h128_step")
    if "cfg2_h256" in which:
        cfg2_wide_case(R, 256, "cfg2_h256_step")


if __name__ == "__main__":
    main()
