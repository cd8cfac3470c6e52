#!/usr/bin/env python
"""Benchmark of the NF-APACT hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3], "cfg4"): 8 independent cfg3 frames
(N=512 transducers, T=4096, 512x512 @ 0.1 mm, K=32 delays, 225 patches of
64x64, SIREN 2->128x4->1), seeds 0-7, sharded over the ranks (frame f on rank
f % N).  A step is one NF-APACT iteration (optimize.hpp:413-471: render ->
wavefronts -> fused Fourier loss -> ray backward -> TV -> SIREN backward ->
Adam) of every frame; `value` is frame-iterations/s over the whole job.
`e2e` runs each frame end to end through the C-ABI (pact_joint_reconstruct,
10 iterations as the cfg4 frame definition of SURVEY §8(d)) from pinned host
signals to a host image.  One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
N_FRAMES = 8
E2E_ITERS = 10
E2E_REPS = 3  # timed joint_reconstruct_batch calls (after one untimed call)
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # FFMA pipe at max clock


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic():
    """Per-launch DRAM bytes of the hot kernels from the committed ncu capture."""
    for name in ("traffic_r02g.json", "traffic_r02f.json", "traffic_r02e.json", "traffic_r02d.json", "traffic_r02.json"):  # the latest committed capture
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)
        except OSError:
            continue
    return {}


def das_physical(traffic):
    """Issue / LSU / shared-memory utilisation of das_stack_kernel<32> at cfg3
    from the committed ncu capture (profiles/traffic_r02g.json)."""
    d = traffic.get("_das_cfg3")
    if not d:
        return None
    wf = d["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]
    return {"issue_active_pct": d["smsp__issue_active.avg.pct_of_peak_sustained_active"],
            "lsu_pipe_pct": d["sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"],
            "fma_pipe_pct": d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"],
            "smem_ld_wavefronts": wf,
            "smem_bank_conflict_frac": d["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"] / wf,
            "source": "ncu --set full, das_stack_kernel<32> at cfg3 (profiles/r02g_das_ncu_raw.csv.gz)"}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def ray_steps(w, cfg):
    """Total midpoint steps of one wavefront pass (make_ray / aberration.hpp:153-171)."""
    from paper_2409_10876_b200.api import make_patch_layout

    lay = make_patch_layout(w.grid, cfg.patch_mm, cfg.overlap)
    c = lay.centers
    th = 2 * np.pi * np.arange(cfg.n_angles) / cfg.n_angles
    ux, uy = np.cos(th)[None, :], np.sin(th)[None, :]
    cx, cy = c[:, :1], c[:, 1:]
    R = w.ring.radius
    b = cx * ux + cy * uy
    cc = cx**2 + cy**2 - R * R
    t_ring = -b + np.sqrt(b * b - cc)
    ex, ey = cx + ux * t_ring, cy + uy * t_ring
    dx, dy = ex - cx, ey - cy
    ln = np.hypot(dx, dy)
    vx, vy = dx / ln, dy / ln
    m = w.mask
    mx, my = cx - m.center_x, cy - m.center_y
    bq = mx * vx + my * vy
    cq = mx * mx + my * my - m.radius**2
    disc = bq * bq - cq
    s = np.sqrt(np.maximum(disc, 0))
    t0 = np.maximum(-bq - s, 0)
    t1 = np.minimum(-bq + s, ln)
    ok = (disc >= 0) & (t0 < t1)
    n = np.where(ok, np.maximum(1, np.ceil((t1 - t0) / cfg.ray_step)), 0)
    return int(n.sum())


def work_model(w, cfg, n_masked):
    """Algorithmic work of one iteration per stage."""
    H, L = cfg.hidden, cfg.sine_layers
    mac_px = 2 * H + (L - 1) * H * H + H
    from paper_2409_10876_b200.api import make_patch_layout

    lay = make_patch_layout(w.grid, cfg.patch_mm, cfg.overlap)
    P = lay.patch_pixels
    steps = ray_steps(w, cfg)
    return {
        "siren_flops": 6.0 * mac_px * n_masked,
        "ray_steps": steps,
        "wavefront_bytes": 16.0 * steps,
        "ray_backward_bytes": 16.0 * steps,
        "fused_loss_bytes": 8.0 * lay.n_patches * len(cfg.delays) * P * P,
    }


# --------------------------------------------------------------------------- #
# CPU reference arm and cpu_baseline leg: the reference's own code
# (oracle/_ref = /root/reference/proj/include compiled unmodified).  Nothing
# here imports the product package: the workload comes from workload_defs.py.
# --------------------------------------------------------------------------- #

WORKLOAD_DESC = ("cfg4: 8 independent cfg3 frames (N=512, T=4096, 512x512 @0.1mm, K=32 in [-2,2] "
                 "mm, 225 patches 64x64, SIREN 2->128x4->1, 512 angles, ray step 0.05 mm)")


def ref_frame_signals(R, w, seed):
    """Frame `seed` of the workload through the reference's simulate_signals
    (phantom.hpp:282-362), rounded to fp32 as the GPU arm's signals are; the
    GPU simulator matches it to <=1e-4 (tests/test_bench_configs_gpu.py)."""
    import workload_defs as wd

    p, sos = wd.phantom_rasters(w, seed)
    return R.simulate(w, p, sos, wd.simulation_mask(w)).astype(np.float32).astype(np.float64)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from types import SimpleNamespace

    import workload_defs as wd
    from oracle_lib import ref

    R = ref()
    if R is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libpact_ref.so not built (make ref)"}))
        return
    w = wd.cfg3()
    cores = os.cpu_count() or 1
    t_all = time.perf_counter()
    sig = ref_frame_signals(R, w, 0)
    t_sim = time.perf_counter() - t_all
    # The stock public entry point, joint_reconstruct (optimize.hpp:367-494),
    # with one step per epoch: LossReport.wall_time of each epoch is exactly
    # one iteration (optimize.hpp:409, 473-474).  The first epoch is the
    # warm-up; the next `steps` epochs are the timed iterations.
    warm = 1
    cfg = SimpleNamespace(**wd.train_fields(w, epochs=warm + args.steps, steps_per_epoch=1,
                                            seed=0, workers=0))
    n_params = R.param_count(w.hidden, w.sine_layers)
    t_jr = time.perf_counter()
    reports, _, _, _ = R.joint_reconstruct(sig, w.ring, w.meta, w.grid, w.mask, cfg, n_params)
    t_jr = time.perf_counter() - t_jr
    step_s = [float(x) for x in reports[warm:, 3]]
    t = sum(step_s)
    value = args.steps / t
    sample = (f"the full cfg3 frame 0 (reference-simulated seed-0 phantom) through the stock "
              f"pact::joint_reconstruct, epochs={warm + args.steps}, steps_per_epoch=1, "
              f"workers={cores} (0 = hardware_concurrency); each timed step is one epoch's "
              f"LossReport.wall_time (one iteration, optimize.hpp:413-471); epoch 1 is the warm-up. "
              f"render_sos / backprop_sos are single-threaded in the reference")
    line = {
        "metric": "NF-APACT iterations/s", "value": value, "unit": "frame-iterations/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "warmup_run": warm, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC,
                   "signals": "straight-ray simulation of seeded phantoms (frame 0 = seed 0; "
                              "reference simulate_signals here)"},
        "cpu_baseline": {"value": value, "unit": "frame-iterations/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "frame-iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "step_seconds": step_s,
        "wall_seconds": {"simulate_signals": t_sim, "joint_reconstruct_call": t_jr,
                         "total": time.perf_counter() - t_all},
        "loss_report_last": {"data_term": float(reports[-1, 0]), "tv_term": float(reports[-1, 1])},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(sig64, n_patch_sample=8):
    """cpu_baseline of our arm (rank 0, N=1): one full reference iteration of
    frame 0 (the same fp32 signals the GPU used) with all host threads, and the
    workers=1 figure of SURVEY §8(d) from the same session.  ~30 s."""
    from types import SimpleNamespace

    import workload_defs as wd
    from oracle_lib import ref

    R = ref()
    if R is None:
        return {"value": None, "unit": "frame-iterations/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref missing on this machine"}
    w = wd.cfg3()
    cores = os.cpu_count() or 1
    cfg = SimpleNamespace(**wd.train_fields(w, seed=0, workers=0))
    h, setup_s = R.nf_session(sig64, w.ring, w.meta, w.grid, w.mask, cfg)
    try:
        full = R.nf_session_step(h, 0)
        one = R.nf_session_step(h, 1, 0, n_patch_sample, with_siren=False)
    finally:
        R.nf_session_close(h)
    n_p = 225
    serial = full["render"] + full["tv"] + full["backprop"] + full["adam"]
    w1 = serial + one["patches"] * n_p / n_patch_sample
    return {"value": 1.0 / full["total"], "unit": "frame-iterations/s", "cores": cores,
            "kind": "reference",
            "sample": (f"one full reference iteration (optimize.hpp:413-467: render_sos, 225 x "
                       f"{{wavefront_profile, fused_patch_loss_grad, wavefront_grad_trace}}, "
                       f"tv_loss, backprop_sos, adam_step) of cfg3 frame 0, workers={cores}, after "
                       f"the one-time DAS + spectra ({setup_s:.1f} s, untimed)"),
            "phases_s": full,
            "workers_1": {"value": 1.0 / w1, "cores": 1,
                          "how": (f"SIREN render + TV + backprop + Adam as measured above (the "
                                  f"reference's SIREN is single-threaded at any worker count) + "
                                  f"the per-patch loop at workers=1 timed on {n_patch_sample} "
                                  f"patches ({one['patches']:.2f} s) x {n_p}/{n_patch_sample}")}}


# --------------------------------------------------------------------------- #
# our arm
# --------------------------------------------------------------------------- #

CFG5_WARMUP, CFG5_STEPS = 2, 5


def cfg5_line(ctx, rank, world, local):
    """BASELINE configs[4] (cfg5: one 2048^2 frame, N=1024, T=8192, K=64, 961
    patches of 128^2, SIREN 2->256x4->1) over the job's ranks: each rank owns
    1/N of the patch rows (and beamforms only their row band) and 1/N of the
    pixels; NCCL all-gather / reduce-scatter / all-reduce between the phases
    (distributed.PartitionedFrame).  ms per full iteration (max over ranks,
    CUDA events) and the DAS of the rank's row band."""
    import torch
    import torch.distributed as dist

    from paper_2409_10876_b200 import workloads as wl
    from paper_2409_10876_b200.api import GridSpec, Trainer
    from paper_2409_10876_b200.distributed import PartitionedFrame, TorchComm

    w = wl.cfg5()
    sig = wl.simulate(ctx, w, seed=0)
    cfg = wl.train_config(w, seed=0)
    tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, cfg,
                 partition=(rank, world) if world > 1 else None)
    info = tr.local()
    frame = PartitionedFrame(tr, TorchComm()) if world > 1 else None

    def step():
        if frame is None:
            tr.step(1)
        else:
            frame.step(1)

    def timed(fn, reps, stream=None):
        # events on the timing stream, joined with the engine's private stream
        # (where the iteration's last phase runs) on both sides
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        if stream is not None:
            stream.wait_event(a)
        for _ in range(reps):
            fn()
        if stream is not None:
            e = torch.cuda.Event()
            e.record(stream)
            cur.wait_event(e)
        b.record(cur)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(CFG5_WARMUP):
        step()
    it_ms = timed(step, CFG5_STEPS, tr.stream())
    data, tv, _ = tr.report(1)
    tr.close()
    # DAS of this rank's row band (the stack rows its patches cover)
    r0, nr = info["stack_row0"], info["stack_rows"]
    g = w.grid
    band = GridSpec(g.width, nr, g.pitch, g.origin_x, g.origin_y + r0 * g.pitch)
    out = torch.empty((len(w.delays), nr, g.width), device="cuda")
    das = lambda: ctx.das_stack(sig, w.ring, w.meta, band, w.v0, w.delays, out=out)  # noqa: E731
    das()
    das_ms = timed(das, 3)
    taps = len(w.delays) * g.width * g.height * w.ring.n_transducers
    return {"workload": "cfg5 (BASELINE configs[4]): 2048x2048 @0.05mm, N=1024, T=8192, K=64 "
                        "in [-3,3] mm, 961 patches 128x128, SIREN 2->256x4->1",
            "ranks": world, "ms_per_iteration": it_ms, "iterations_per_s": 1e3 / it_ms,
            "steps": CFG5_STEPS, "warmup": CFG5_WARMUP,
            "collectives": ("all_gather dv, reduce_scatter dL/dv (overlapping TV), all_reduce "
                            "report/flags/gradient (NCCL)") if world > 1 else "none (one rank)",
            "das_band_rows": nr, "das_ms": das_ms,
            "das_gsamples_per_s": taps * (nr / g.height) * world / (das_ms * 1e-3) / 1e9,
            "loss_report": {"data_term": data, "tv_term": tv}}


def run_ours(args):
    # a stuck run leaves the Python stacks on stderr (every 10 minutes)
    import faulthandler
    faulthandler.dump_traceback_later(600, repeat=True)
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2409_10876_b200 import _abi
    from paper_2409_10876_b200 import workloads as wl
    from paper_2409_10876_b200.api import Context, SirenSpec, Trainer, joint_reconstruct_batch

    w = wl.cfg3()
    cfg = wl.train_config(w)
    ctx = Context(local)
    L = _abi.lib()
    my_frames = wl.shard_frames(N_FRAMES, rank, world)
    hbm, bf16, peak_src = peaks()

    # ---- inputs: simulated on the GPU from seeded phantoms (one-time) ----
    signals = {f: wl.simulate(ctx, w, seed=f) for f in my_frames}
    torch.cuda.synchronize()

    # ---- DAS stack on its own (the one-time part-1 kernel) ----
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
    stack = torch.empty((len(w.delays), w.grid.height, w.grid.width), device="cuda")
    s0 = signals[my_frames[0]]
    for _ in range(3):
        ctx.das_stack(s0, w.ring, w.meta, w.grid, w.v0, w.delays, out=stack)
    das_ms = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.das_stack(s0, w.ring, w.meta, w.grid, w.v0, w.delays, out=stack)
        b.record()
        torch.cuda.synchronize()
        das_ms.append(a.elapsed_time(b))
    das_t = statistics.median(das_ms)
    das_ach = w.das_bytes / (das_t * 1e-3) / 1e9
    del stack

    # ---- engines: one trainer per frame (DAS + spectra + init, one-time) ----
    trainers = [Trainer(ctx, signals[f], w.ring, w.meta, w.grid, w.mask,
                        wl.train_config(w, seed=f)) for f in my_frames]
    torch.cuda.synchronize()
    n_masked = int(L.pact_masked_count(C.byref(w.grid.c()), C.byref(w.mask.c())))
    work = work_model(w, cfg, n_masked)

    def step_all():
        for tr in trainers:
            tr.step(1)

    clk = Clocks(local).start()
    for _ in range(max(3, args.warmup)):
        step_all()
    torch.cuda.synchronize()
    # eager iterations with per-stage events; per-stage median of five (a
    # single sample moves by 10 % with the box's power state)
    samples = [trainers[0].profile_step() for _ in range(5)]
    stages = {k: statistics.median(smp[k] for smp in samples) for k in samples[0]}
    torch.cuda.synchronize()

    # ---- timed region: K iterations of every frame, frames on their own streams ----
    tstream = torch.cuda.current_stream()
    streams = [tr.stream() for tr in trainers]
    n0 = sum(tr.launch_count() for tr in trainers)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(tstream)
    for s in streams:
        s.wait_event(start)
    for _ in range(args.steps):
        step_all()
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        tstream.wait_event(e)
    end.record(tstream)
    torch.cuda.synchronize()
    clk.stop()
    launches = sum(tr.launch_count() for tr in trainers) - n0
    if world > 1:
        dist.barrier()
    t_ms = torch.tensor([start.elapsed_time(end)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    total_ms = float(t_ms.item())
    value = N_FRAMES * args.steps / (total_ms * 1e-3)
    reports = [tr.report() for tr in trainers]
    for tr in trainers:
        tr.close()
    del trainers

    # ---- end to end: pinned host signals -> joint_reconstruct_batch -> host image ----
    # the public batch entry point runs this rank's frames concurrently (one
    # engine stream each), exactly as separate joint_reconstruct calls would
    # compute them; H2D of every frame's signals and D2H of every image + SOS
    # are inside the timed region
    nbytes_in = w.ring.n_transducers * w.meta.n_samples * 4
    nbytes_out = 2 * w.grid.width * w.grid.height * 4
    hin = {f: torch.empty(signals[f].shape, dtype=torch.float32, pin_memory=True) for f in my_frames}
    for f in my_frames:
        hin[f].copy_(signals[f])
    hout = {f: torch.empty((2, w.grid.height, w.grid.width), dtype=torch.float32, pin_memory=True)
            for f in my_frames}
    e2e_cfgs = [wl.train_config(w, epochs=E2E_ITERS, steps_per_epoch=1, seed=f) for f in my_frames]
    del signals
    def e2e_call():
        # host buffers straight through the C-ABI: the library uploads each
        # frame's signals and downloads its image + SOS on the frame's stream
        joint_reconstruct_batch(ctx, [hin[f] for f in my_frames], w.ring, w.meta, w.grid, w.mask,
                                e2e_cfgs, images=[hout[f][0] for f in my_frames],
                                sos=[hout[f][1] for f in my_frames])

    e2e_call()  # untimed: first-call costs (cuFFT plans, pool growth, module load)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(E2E_REPS):
        e2e_call()
    b.record()
    torch.cuda.synchronize()
    e2e_t = torch.tensor([a.elapsed_time(b)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = N_FRAMES * E2E_ITERS * E2E_REPS / (float(e2e_t.item()) * 1e-3)

    # ---- per-stage roofline of one frame-iteration ----
    siren_ms = stages["siren_fwd"] + stages["siren_bwd"]
    stage_rl = {
        "siren_fwd+bwd": {"ms": siren_ms, "achieved_tflops": work["siren_flops"] / (siren_ms * 1e-3) / 1e12},
        "wavefront": {"ms": stages["wavefront"],
                      "achieved_gbs": work["wavefront_bytes"] / (stages["wavefront"] * 1e-3) / 1e9},
        "ray_backward": {"ms": stages["ray_backward"],
                         "achieved_gbs": work["ray_backward_bytes"] / (stages["ray_backward"] * 1e-3) / 1e9},
        "fused_loss": {"ms": stages["fused_loss"],
                       "achieved_gbs": work["fused_loss_bytes"] / (stages["fused_loss"] * 1e-3) / 1e9},
        "tv_report": {"ms": stages["tv_report"]}, "adam": {"ms": stages["adam"]},
    }
    traffic = load_traffic()
    sr = stage_rl["siren_fwd+bwd"]
    # the width-128 SIREN GEMMs (forward chain and fused backward) run on the
    # tensor cores with split-fp16 operands (three kind::f16 MMAs per
    # fp32-accurate product): the ceiling is a third of the dense 16-bit rate
    # (= the measured bf16 rate); 3xTF32 (the PACT_SIREN_F16=0 /
    # PACT_SIREN_BWD_F16=0 variants, and cfg5's width-256 layers) is half that
    f16x3 = bf16 / 3.0
    tf32x3 = bf16 / 2.0 / 3.0
    sr["bf16_dense_peak_tflops"] = bf16
    sr["tensor_split_f16_peak_tflops"] = f16x3
    sr["frac_of_split_f16_tensor"] = sr["achieved_tflops"] / f16x3
    sr["tensor_3xtf32_peak_tflops"] = tf32x3
    sr["fp32_pipe_peak_tflops"] = FP32_PEAK_TFLOPS  # the SIMT path's ceiling, for reference
    # The roofline line is for the dominant kernel.  Since the ray adjoint
    # became a gather (round 2) the SIREN is the largest stage; its forward is
    # ONE persistent tcgen05 kernel (siren_chain_pair_kernel: every layer of
    # every pixel tile, two tiles in flight), so the line is that kernel
    # against its tensor ceiling: split-fp16 operands, three kind::f16 MMAs per
    # fp32-accurate product at the dense 16-bit rate (= the measured bf16
    # rate), i.e. a third of it.  The ray stages are L1/texture-served (their
    # 16 B/step model exceeds HBM) and are reported per stage.
    fwd_flops = work["siren_flops"] / 3.0  # 2 FLOP per MAC, forward only
    fwd_ach = fwd_flops / (stages["siren_fwd"] * 1e-3) / 1e12
    roofline = {"bound": "tensor", "achieved": fwd_ach, "peak": f16x3, "unit": "TFLOP/s",
                "frac": fwd_ach / f16x3, "traffic": traffic.get("siren_chain_pair_kernel"),
                "kernel": "siren_chain_pair_kernel",
                "peak_source": f"measured dense bf16 {bf16:.1f} TFLOP/s / 3 (split fp16: three "
                               f"kind::f16 MMAs per fp32-accurate product at the dense 16-bit rate)",
                "work_model": "SURVEY 8(d): 2 FLOP per MAC of the 2->128x4->1 network per masked "
                              "pixel (fp32-equivalent FLOPs)",
                "traffic_source": traffic.get("_source")}
    # SURVEY 8(d) iteration roofline: sum_k max(B_k / HBM, F_k / peak_k), SIREN at split fp16
    # the loss reads half of Y since round 2b (the real stack's Hermitian
    # spectrum): its model bytes stay the full read, like SURVEY 8(d)
    model_ms = 1e3 * (work["siren_flops"] / (f16x3 * 1e12)
                      + (work["wavefront_bytes"] + work["ray_backward_bytes"]
                         + work["fused_loss_bytes"]) / (hbm * 1e9))
    iter_ms = sum(v["ms"] for v in stage_rl.values())
    iteration_roofline = {"model_ms": model_ms, "measured_ms": iter_ms, "frac": model_ms / iter_ms,
                          "model": "SURVEY 8(d): SIREN forward and backward F at the split-fp16 "
                                   "tensor rate (measured dense bf16 / 3), ray and loss "
                                   "algorithmic bytes at measured HBM; "
                                   "measured = sum of stage CUDA-event times of one frame. frac > 1: "
                                   "the ray stages are L1/texture-served, below their HBM byte model"}

    cfg5 = None
    if not args.no_cfg5:
        torch.cuda.empty_cache()
        try:
            cfg5 = cfg5_line(ctx, rank, world, local)
        except Exception as e:  # the headline numbers above stand without the cfg5 extra
            cfg5 = {"error": f"{type(e).__name__}: {e}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_leg(hin[my_frames[0]].double().numpy())

    if rank == 0:
        line = {
            "metric": "NF-APACT iterations/s", "value": value, "unit": "frame-iterations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD_DESC,
                       "frames_on_rank0": len(my_frames),
                       "signals": "straight-ray simulation of seeded phantoms (seeds 0-7; "
                                  "pact_simulate_signals here)",
                       "l2": "per-frame working set (Y 236 MB + activations 537 MB) > 126 MB L2",
                       "parallelism": f"{world} rank(s), frames sharded f % N, one CUDA stream per frame"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": "frame-iterations/s",
                    "h2d_bytes_per_step": nbytes_in * N_FRAMES // world,
                    "d2h_bytes_per_step": nbytes_out * N_FRAMES // world,
                    "what": f"all frames of the rank: pact_joint_reconstruct_batch on pinned HOST "
                            f"buffers (per frame, on its own stream: H2D signals, DAS, spectra, "
                            f"{E2E_ITERS} iterations, final deconvolution, D2H image+SOS; frames "
                            f"concurrent); {E2E_REPS} timed calls after one untimed call (bytes are "
                            f"per call)"},
            "gpu_launches": launches,
            "roofline": roofline,
            "iteration_roofline": iteration_roofline,
            "stages_ms_one_frame": stage_rl,
            "das": {"ms": das_t, "gsamples_per_s": w.das_samples / (das_t * 1e-3) / 1e9,
                    "roofline": {"bound": "hbm", "achieved": das_ach, "peak": hbm, "unit": "GB/s",
                                 "frac": das_ach / hbm, "peak_source": peak_src,
                                 "byte_model": "8*S + 4*K*W*H + 4*N*T, S = W*H*K*N"},
                    # the physically binding limits: taps are served from
                    # shared memory, so issue slots and the LSU pipe bound the kernel
                    "physical": das_physical(traffic)},
            "loss_report_frame0": reports[0],
            "cfg5": cfg5,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def dry_run(args):
    """The N-rank launch path without GPU work: every rank joins a gloo group,
    the ranks agree on the world size, and rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([rank], dtype=torch.int64)
        dist.all_reduce(t)
        assert int(t.item()) == world * (world - 1) // 2
        dist.barrier()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "requested": args.gpus,
                          "impl": args.impl}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` run without torchrun: launch N ranks (one per GPU)
    the way the driver does, over 127.0.0.1; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check only: join the ranks over gloo and print one line")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    _, world, _ = dist_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        dry_run(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
