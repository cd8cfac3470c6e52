"""One NF-APACT frame over several GPUs: the phase
orchestration of a partitioned trainer with its collectives.

Each rank creates `Trainer(..., partition=(rank, world))` (patch rows, their
DAS row band, and a contiguous share of the masked pixels, see
pact_trainer_create_partitioned) and calls `PartitionedFrame.step()`; between
the library's phases the ranks exchange over NCCL (NVLink/NVSwitch) through
torch.distributed.  When the pixel shares are equal raster slabs (the mask
covers the grid and the rank count divides it — cfg5: 2048^2 / 8), the
exchanges are the minimal ones:

    phase 0 render own pixels          -> all_gather(dv)             4·H·W/N out per rank
    phase 6 wavefronts, loss, rays     -> reduce_scatter(dL/dv)      8·H·W/N in per rank
    phase 7 TV, report  (overlaps the reduce-scatter)
                                       -> all_reduce(report SUM, flags MAX)
    phase 2 SIREN backward (own slab)  -> all_reduce(grad, SUM)      8·P bytes
    phase 3 Adam (replicated)

otherwise dv and dL/dv are all-reduced (SUM; each pixel has one owner).
Every rank ends each step with the same theta (the gradient is identical
after the all-reduce, Adam runs on each replica), so there is no parameter
broadcast.  The collectives run on the caller's current stream, ordered
against the engine's private stream with stream waits (no host syncs).

`comm` is anything with `all_reduce(t, op)`, `all_gather(out, inp)`,
`reduce_scatter(out, inp)` and `SUM` / `MAX` attributes: `TorchComm`
(torch.distributed) for real runs, or a test double.
"""
from __future__ import annotations

import torch

from .api import Trainer


class TorchComm:
    """torch.distributed collectives, ordered on the caller's current stream.
    NCCL runs all-gather / reduce-scatter in place (the slab is a view of the
    full raster); gloo (CPU tests) has no tensor reduce-scatter, so it is an
    all-reduce plus the slab copy there."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.SUM, self.MAX = dist.ReduceOp.SUM, dist.ReduceOp.MAX
        self.nccl = dist.get_backend(group) == "nccl"

    def all_reduce(self, t: torch.Tensor, op):
        self.dist.all_reduce(t, op=op, group=self.group)

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor):
        if self.nccl:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
        else:
            parts = list(out.chunk(self.dist.get_world_size(self.group)))
            self.dist.all_gather(parts, inp.clone(), group=self.group)

    def reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor):
        if self.nccl:
            self.dist.reduce_scatter_tensor(out, inp, op=self.SUM, group=self.group)
        else:
            full = inp.clone()
            self.dist.all_reduce(full, op=self.SUM, group=self.group)
            r = self.dist.get_rank(self.group)
            out.copy_(full.chunk(self.dist.get_world_size(self.group))[r])


class PartitionedFrame:
    """Drives one partitioned trainer of a multi-GPU frame."""

    def __init__(self, trainer: Trainer, comm):
        self.tr, self.comm = trainer, comm
        g = trainer.grid
        H, W = g.height, g.width
        self.dv = trainer.view(2, (H, W), torch.float32)
        self.gv = trainer.view(5, (H, W), torch.float64)
        self.grad = trainer.view(6, (trainer.n_params,), torch.float64)
        self.report = trainer.view(8, (3,), torch.float64)
        self.flags = trainer.view(9, (1,), torch.int32)
        self.num = self.den = None
        info = trainer.local()
        world, rank = info["world"], info["rank"]
        if world > 1:
            self.num = trainer.view(10, (H, W), torch.float32)
            self.den = trainer.view(11, (H, W), torch.float32)
        # equal raster slabs: pixel share r = rows-major pixels [r npx/N, (r+1) npx/N)
        npx = H * W
        self.slab = None
        if (world > 1 and getattr(trainer, "n_masked", None) == npx and npx % world == 0
                and info.get("pixel_lo") == rank * npx // world
                and info.get("pixel_hi") == (rank + 1) * npx // world):
            self.slab = (rank * npx // world, (rank + 1) * npx // world)
        self.engine = trainer.stream()

    def _comm_stream(self):
        cur = torch.cuda.current_stream() if self.engine is not None else None
        if cur is not None:
            cur.wait_stream(self.engine)
        return cur

    def _join(self, cur):
        if cur is not None:
            self.engine.wait_stream(cur)

    def _reduce(self, *pairs):
        cur = self._comm_stream()
        for t, op in pairs:
            self.comm.all_reduce(t, op)
        self._join(cur)

    def _share_dv(self):
        if self.slab is None:
            self._reduce((self.dv, self.comm.SUM))
            return
        cur = self._comm_stream()
        flat = self.dv.view(-1)
        lo, hi = self.slab
        self.comm.all_gather(flat, flat[lo:hi])
        self._join(cur)

    def step(self, n: int = 1):
        c = self.comm
        for _ in range(n):
            self.tr.phase(0)
            self._share_dv()
            self.tr.phase(6)
            # dL/dv to its owners while the engine runs TV + the report
            cur = self._comm_stream()
            if self.slab is None:
                c.all_reduce(self.gv, c.SUM)
            else:
                flat = self.gv.view(-1)
                lo, hi = self.slab
                c.reduce_scatter(flat[lo:hi], flat)
            self.tr.phase(7)
            if cur is not None:
                cur.wait_stream(self.engine)
            c.all_reduce(self.report, c.SUM)
            c.all_reduce(self.flags, c.MAX)
            self._join(cur)
            self.tr.phase(2)
            self._reduce((self.grad, c.SUM))
            self.tr.phase(3)

    def finish(self):
        """The final image and SOS (optimize.hpp:478-486) of the whole frame,
        on every rank: fp32 [H, W] each."""
        c = self.comm
        self.tr.phase(4)
        self._share_dv()
        v0 = self.tr.v0
        if self.num is None:  # world == 1
            return self.tr.finish()
        self.tr.phase(5)
        self._reduce((self.num, c.SUM), (self.den, c.SUM))
        img = torch.where(self.den > 0, self.num / self.den, torch.zeros_like(self.num))
        return img, self.dv + v0
