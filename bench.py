#!/usr/bin/env python
"""Benchmark of the NF-APACT hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  For N > 1 the driver launches one process per GPU
with torchrun; ranks shard independent units (weak scaling) and the timed
region is bracketed by barrier + synchronize, max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
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
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
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


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------------------- #
# CPU reference arm: the reference's own das_stack (oracle/_ref), all threads
# --------------------------------------------------------------------------- #

def ref_das_seconds(w, sig64, reps, workers):
    from oracle_lib import REF_PATH

    L = C.CDLL(REF_PATH)
    f = L.ref_time_das_stack
    _D, _I, _P = C.c_double, C.c_int, C.c_void_p
    f.argtypes = [_I, _I, _D, _D, _I, _D, _D, _P, _I, _I, _D, _D, _D, _D, _I, _P, _I]
    f.restype = C.c_double
    d = np.ascontiguousarray(w.delays, dtype=np.float64)
    g = w.grid
    return f(reps, w.ring.n_transducers, w.ring.radius, w.ring.angle_offset, w.meta.n_samples,
             w.meta.dt, w.meta.t0, sig64.ctypes.data_as(_P), g.width, g.height, g.pitch,
             g.origin_x, g.origin_y, w.v0, len(d), d.ctypes.data_as(_P), workers)


def cpu_slab(w, rows):
    """A row slab of the workload's grid (bounded CPU sample)."""
    from paper_2409_10876_b200.api import GridSpec
    from dataclasses import replace

    g = w.grid
    y0 = (g.height - rows) // 2
    slab = GridSpec(g.width, rows, g.pitch, g.origin_x, g.origin_y + y0 * g.pitch)
    return replace(w, grid=slab)


def run_reference(args):
    rank, world, _ = dist_env()
    from paper_2409_10876_b200 import workloads as wl

    w = wl.cfg3()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    sig = wl.iid_signals(w, 0).astype(np.float64)
    # bounded sample: a 64-row slab of the cfg3 grid (1/8 of the taps)
    slab = cpu_slab(w, 64)
    frac = slab.das_samples / w.das_samples
    for _ in range(args.warmup):
        ref_das_seconds(slab, sig, 1, cores)
    secs = [ref_das_seconds(slab, sig, 1, cores) for _ in range(args.steps)]
    t = sum(secs)
    value = args.steps * slab.das_samples / t / 1e9
    line = {
        "metric": "DAS-stack GSamples/s", "value": value, "unit": "GSamples/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps / frac, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 DAS stack (N=512, T=4096, 512x512, K=32)",
                   "signals": "iid N(0,1) seed 0", "sample": "64-row slab of the grid per step"},
        "cpu_baseline": {"value": value, "unit": "GSamples/s", "cores": cores,
                         "kind": "reference",
                         "sample": "das_stack on a 64x512-pixel slab (1/8 of cfg3) per step"},
        "e2e": {"value": value, "unit": "GSamples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- #
# our arm
# --------------------------------------------------------------------------- #

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2409_10876_b200 import _abi
    from paper_2409_10876_b200 import workloads as wl
    from paper_2409_10876_b200.api import Context

    w = wl.cfg3()
    ctx = Context(local)
    stream = torch.cuda.current_stream()
    L = _abi.lib()

    # Each rank beamforms its own frame (seed = rank): independent units.
    sig_h = wl.iid_signals(w, rank)
    sig = torch.as_tensor(sig_h).cuda()
    K, H, W = len(w.delays), w.grid.height, w.grid.width
    out = torch.empty((K, H, W), device="cuda", dtype=torch.float32)
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)

    def step():
        ctx.das_stack(sig, w.ring, w.meta, w.grid, w.v0, w.delays, out=out)

    clk = Clocks(local).__enter__()  # sampling starts with the warm-up load
    t_w = time.time()
    n_warm = 0
    while n_warm < max(3, args.warmup) or time.time() - t_w < 0.5:
        step()
        n_warm += 1
        if n_warm % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = ctx.launch_count()
    for i in range(args.steps):
        flush.zero_()  # L2 flush (256 MB > 126 MB L2) outside the event pair
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    clk.__exit__()
    launches = ctx.launch_count() - n0
    if world > 1:
        dist.barrier()
    ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = torch.tensor([sum(ms)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    total_ms = float(t_ms.item())
    per_step_ms = total_ms / args.steps
    value = world * w.das_samples * args.steps / (total_ms * 1e-3) / 1e9

    # ---- end-to-end through the C-ABI with host buffers ----
    nbytes_in = sig_h.nbytes
    nbytes_out = K * H * W * 4
    hin = C.c_void_p()
    hout = C.c_void_p()
    _abi.check(L.pact_host_alloc_pinned(nbytes_in, C.byref(hin)))
    _abi.check(L.pact_host_alloc_pinned(nbytes_out, C.byref(hout)))
    C.memmove(hin, sig_h.ctypes.data, nbytes_in)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        a.record(stream)
        _abi.check(L.pact_upload(ctx.handle, C.c_void_p(sig.data_ptr()), hin, nbytes_in))
        step()
        _abi.check(L.pact_download(ctx.handle, hout, C.c_void_p(out.data_ptr()), nbytes_out))
        b.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    e2e_t = torch.tensor([sum(e2e_ms)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world * w.das_samples * args.steps / (float(e2e_t.item()) * 1e-3) / 1e9
    L.pact_host_free_pinned(hin)
    L.pact_host_free_pinned(hout)

    # ---- roofline of the dominant kernel (DAS) ----
    hbm, src = peaks()
    achieved = w.das_bytes / (per_step_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None,
                "peak_source": src,
                "byte_model": "8*S + 4*K*W*H + 4*N*T (SURVEY 8(d)), S = W*H*K*N"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle_lib import REF_PATH

        if os.path.exists(REF_PATH):
            cores = os.cpu_count() or 1
            slab = cpu_slab(w, 32)
            secs = ref_das_seconds(slab, sig_h.astype(np.float64), 1, cores)
            cpu = {"value": slab.das_samples / secs / 1e9, "unit": "GSamples/s",
                   "cores": cores, "kind": "reference",
                   "sample": f"reference das_stack on a 32-row slab of cfg3 ({secs:.1f} s)"}
        else:
            cpu = {"value": None, "unit": "GSamples/s", "cores": 0, "kind": "reference",
                   "sample": "oracle/_ref missing on this machine"}

    if rank == 0:
        line = {
            "metric": "DAS-stack GSamples/s", "value": value, "unit": "GSamples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": per_step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg3 DAS stack (N=512, T=4096, 512x512 @0.1mm, K=32 in [-2,2] mm)",
                       "signals": "iid N(0,1), seed = rank", "l2": "flushed (256 MB write) between steps",
                       "parallelism": f"{world} independent frames"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": "GSamples/s", "h2d_bytes_per_step": nbytes_in,
                    "d2h_bytes_per_step": nbytes_out},
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
