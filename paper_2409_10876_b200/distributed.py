"""One NF-APACT frame over several GPUs: the phase
orchestration of a partitioned trainer with its collectives.

Each rank creates `Trainer(..., partition=(rank, world))` (patch rows and a
contiguous share of the masked pixels, see pact_trainer_create_partitioned)
and calls `PartitionedFrame.step()`; between the library's phases the ranks
all-reduce, over NCCL (NVLink/NVSwitch) through torch.distributed:

    phase 0 render own pixels          -> all_reduce(dv,   SUM)  4·H·W bytes
    phase 1 rays, loss, TV, report     -> all_reduce(dL/dv SUM)  8·H·W bytes
                                          all_reduce(report SUM), (flags MAX)
    phase 2 SIREN backward             -> all_reduce(grad, SUM)  8·P bytes
    phase 3 Adam (replicated)

cfg5 per step: 16 MB + 32 MB + 1.6 MB.  Every rank ends each step with the
same theta (the gradient is identical after the all-reduce, Adam runs on each
replica), so there is no parameter broadcast.  The collectives are ordered
against the engine's private stream with stream waits (no host syncs).

`comm` is anything with `all_reduce(tensor, op)` and `SUM` / `MAX`
attributes: `TorchComm` (torch.distributed) for real runs, or a test double.
"""
from __future__ import annotations

import torch

from .api import Trainer


class TorchComm:
    """torch.distributed collectives, ordered on the caller's current stream."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.SUM, self.MAX = dist.ReduceOp.SUM, dist.ReduceOp.MAX

    def all_reduce(self, t: torch.Tensor, op):
        self.dist.all_reduce(t, op=op, group=self.group)


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
        if trainer.local()["world"] > 1:
            self.num = trainer.view(10, (H, W), torch.float32)
            self.den = trainer.view(11, (H, W), torch.float32)
        self.engine = trainer.stream()

    def _reduce(self, *pairs):
        # the collectives run on the current stream after the engine's work,
        # and the engine's next phase waits for them (engine None: host tensors)
        if self.engine is None:
            for t, op in pairs:
                self.comm.all_reduce(t, op)
            return
        cur = torch.cuda.current_stream()
        cur.wait_stream(self.engine)
        for t, op in pairs:
            self.comm.all_reduce(t, op)
        self.engine.wait_stream(cur)

    def step(self, n: int = 1):
        c = self.comm
        for _ in range(n):
            self.tr.phase(0)
            self._reduce((self.dv, c.SUM))
            self.tr.phase(1)
            self._reduce((self.gv, c.SUM), (self.report, c.SUM), (self.flags, c.MAX))
            self.tr.phase(2)
            self._reduce((self.grad, c.SUM))
            self.tr.phase(3)

    def finish(self):
        """The final image and SOS (optimize.hpp:478-486) of the whole frame,
        on every rank: fp32 [H, W] each."""
        c = self.comm
        self.tr.phase(4)
        self._reduce((self.dv, c.SUM))
        v0 = self.tr.v0
        if self.num is None:  # world == 1
            return self.tr.finish()
        self.tr.phase(5)
        self._reduce((self.num, c.SUM), (self.den, c.SUM))
        img = torch.where(self.den > 0, self.num / self.den, torch.zeros_like(self.num))
        return img, self.dv + v0
