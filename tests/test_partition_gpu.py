"""One frame split over ranks (SURVEY §8(e), cfg5 design) on one GPU.

A partitioned trainer owns patch rows and a share of the masked pixels; the
ranks all-reduce dv, dL/dv, the report/flags and the gradient between phases
(distributed.PartitionedFrame over NCCL).  Here the ranks run in one process
and the all-reduces are tensor sums, which checks the partition itself:
  * world = 1 driven by phases is bitwise the fused (graph) step;
  * world = 2 / 4 reproduces the single-rank iteration (reports, theta, final
    image and SOS) up to the summation order of the split reductions.
"""
from dataclasses import replace

import numpy as np
import pytest
import torch

import golden_util as gu
from oracle_lib import rel_l2
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import Trainer
from paper_2409_10876_b200.distributed import PartitionedFrame

pytestmark = pytest.mark.gpu


class _NoComm:
    SUM, MAX = "sum", "max"

    def all_reduce(self, t, op):  # world == 1
        pass


def test_world1_phases_equal_fused_step(ctx):
    G = gu.load("small_instance")
    si = gu.small_instance()
    cfg = replace(si.cfg, seed=3, use_cuda_graph=True)
    sig = torch.as_tensor(G["sig"]).cuda()
    meta = gu.meta(G["meta"])
    a = Trainer(ctx, sig, si.ring, meta, si.grid, si.mask, cfg)
    b = Trainer(ctx, sig, si.ring, meta, si.grid, si.mask, cfg, partition=(0, 1))
    fb = PartitionedFrame(b, _NoComm())
    a.step(3)
    fb.step(3)
    assert a.report(1) == b.report(1)
    assert np.array_equal(a.theta(), b.theta())
    ia, sa = a.finish()
    ib, sb = fb.finish()
    assert torch.equal(ia, ib) and torch.equal(sa, sb)
    a.close()
    b.close()


def _emulated(ctx, sig, w, cfg, world, steps):
    trs = [Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, cfg, partition=(r, world))
           for r in range(world)]
    frames = [PartitionedFrame(t, _NoComm()) for t in trs]

    def reduce(name, op="sum"):
        torch.cuda.synchronize()
        ts = [getattr(f, name) for f in frames]
        acc = ts[0].clone()
        for t in ts[1:]:
            acc = acc + t if op == "sum" else torch.maximum(acc, t)
        for t in ts:
            t.copy_(acc)
        torch.cuda.synchronize()

    for _ in range(steps):
        for f in frames:
            f.tr.phase(0)
        reduce("dv")
        for f in frames:
            f.tr.phase(1)
        reduce("gv")
        reduce("report")
        reduce("flags", "max")
        for f in frames:
            f.tr.phase(2)
        reduce("grad")
        for f in frames:
            f.tr.phase(3)
    torch.cuda.synchronize()
    reps = [t.report(1) for t in trs]
    thetas = [t.theta() for t in trs]
    for f in frames:
        f.tr.phase(4)
    reduce("dv")
    for f in frames:
        f.tr.phase(5)
    reduce("num")
    reduce("den")
    f = frames[0]
    img = torch.where(f.den > 0, f.num / f.den, torch.zeros_like(f.num))
    sos = f.dv + w.v0
    infos = [t.local() for t in trs]
    for t in trs:
        t.close()
    return reps, thetas, img, sos, infos


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_frame_matches_single_rank(ctx, world):
    w = wl.cfg2()
    cfg = replace(wl.train_config(w, seed=1), use_cuda_graph=False)
    sig = wl.simulate(ctx, w, seed=0)
    ref = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, cfg)
    steps = 3
    ref.step(steps)
    want_rep, want_th = ref.report(1), ref.theta()
    want_img, want_sos = ref.finish()
    K, H, W = len(w.delays), w.grid.height, w.grid.width
    full_stack = ref.read(0, (K, H, W), np.float32)
    ref.close()
    # the row-tile DAS split: each rank beamforms only the rows
    # its patch rows cover, and those rows equal the full stack's bit for bit
    bands = []
    for r in range(world):
        t = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, cfg, partition=(r, world))
        info = t.local()
        r0, nr = info["stack_row0"], info["stack_rows"]
        assert 0 < nr < H
        band = t.read(0, (K, nr, W), np.float32)
        assert np.array_equal(band, full_stack[:, r0:r0 + nr])
        bands.append((r0, nr))
        t.close()
    assert bands[0][0] == 0 and bands[-1][0] + bands[-1][1] == H
    reps, thetas, img, sos, infos = _emulated(ctx, sig, w, cfg, world, steps)
    # the partition covers everything exactly once
    assert infos[0]["patch_lo"] == 0 and infos[-1]["patch_hi"] == infos[0]["n_patches"]
    for a, b in zip(infos, infos[1:]):
        assert a["patch_hi"] == b["patch_lo"] and a["pixel_hi"] == b["pixel_lo"]
    # every rank holds the same replica
    for r in range(1, world):
        assert reps[r] == reps[0]
        assert np.array_equal(thetas[r], thetas[0])
    np.testing.assert_allclose(reps[0], want_rep, rtol=1e-6)
    assert rel_l2(thetas[0], want_th) <= 1e-6
    assert rel_l2(sos.double().cpu().numpy() - w.v0, want_sos.double().cpu().numpy() - w.v0) <= 1e-5
    assert rel_l2(img.double().cpu().numpy(), want_img.double().cpu().numpy()) <= 1e-5


def test_world1_nccl_step_equals_fused_step(ctx):
    """The library's own NCCL orchestration (pact_ctx_attach_nccl +
    pact_trainer_step_nccl / finish_nccl, no host framework) on a one-rank
    communicator: bitwise the fused (graph) step and the single-GPU finish.
    More ranks need more GPUs (ranks whose kernels wait on one another must
    not share a GPU); the orchestration is the same code for any world."""
    from paper_2409_10876_b200.api import Context

    G = gu.load("small_instance")
    si = gu.small_instance()
    cfg = replace(si.cfg, seed=3, use_cuda_graph=True)
    sig = torch.as_tensor(G["sig"]).cuda()
    meta = gu.meta(G["meta"])
    c1 = Context(0)
    c1.attach_nccl(Context.nccl_unique_id(), 0, 1)
    a = Trainer(ctx, sig, si.ring, meta, si.grid, si.mask, cfg)
    b = Trainer(c1, sig, si.ring, meta, si.grid, si.mask, cfg, partition=(0, 1))
    a.step(3)
    b.step_nccl(3)
    assert a.report(1) == b.report(1)
    assert np.array_equal(a.theta(), b.theta())
    ia, sa = a.finish()
    ib, sb = b.finish_nccl()
    torch.cuda.synchronize()
    assert torch.equal(ia, ib) and torch.equal(sa, sb)
    a.close()
    b.close()
    c1.close()
