"""The multi-GPU frame orchestration (distributed.PartitionedFrame) over a real
process group: world_size 2 on CPU with gloo, the library trainer replaced by
a host double that records its phases and fills its buffers like a partition
would (each rank owns a share of the pixels, patches and gradient terms).
Checks the collective semantics (SUM for dv / dL/dv / report / gradient and the
final merge accumulators, MAX for the flags) and the phase order, for both
pixel-share forms: interleaved rows (all-reduces) and equal raster slabs
(all-gather of dv, reduce-scatter of dL/dv to the slab owners).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_10876_b200.distributed import PartitionedFrame, TorchComm

H, W, NP = 6, 5, 7


class FakeTrainer:
    """Host stand-in with the Trainer surface PartitionedFrame uses."""

    class _G:
        height, width = H, W

    def __init__(self, rank, world, slab=False):
        self.rank, self.world, self.slab = rank, world, slab
        self.n_masked = H * W
        self.grid = self._G()
        self.n_params = NP
        self.v0 = 1500.0
        self.bufs = {2: torch.zeros(H, W), 5: torch.zeros(H, W, dtype=torch.float64),
                     6: torch.zeros(NP, dtype=torch.float64),
                     8: torch.zeros(3, dtype=torch.float64),
                     9: torch.zeros(1, dtype=torch.int32), 10: torch.zeros(H, W),
                     11: torch.zeros(H, W)}
        self.log = []
        self.seen = {}

    def view(self, what, shape, dtype):
        return self.bufs[what]

    def stream(self):
        return None

    def local(self):
        info = {"world": self.world, "rank": self.rank}
        if self.slab:  # equal raster slabs: H * W = 30 pixels, 15 per rank
            n = H * W // self.world
            info.update(pixel_lo=self.rank * n, pixel_hi=(self.rank + 1) * n)
        return info

    def _own(self, t, value):
        t.zero_()
        if self.slab:
            n = H * W // self.world
            t.view(-1)[self.rank * n:(self.rank + 1) * n] = value
        else:
            t[self.rank::self.world] = value

    def phase(self, k):
        self.log.append(k)
        r = self.rank
        if k == 0:  # own pixels of dv
            self._own(self.bufs[2], 1.0 + r)
        elif k == 6:  # wavefronts, loss, ray adjoint
            self.seen["dv"] = self.bufs[2].clone()
            self.bufs[5].fill_(0.5 * (r + 1))
        elif k == 7:  # TV + report
            self.bufs[8][:] = torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64) * (r + 1)
            self.bufs[9][0] = 4 if r == 1 else 1
        elif k == 2:
            self.seen["gv"] = self.bufs[5].clone()
            self.seen["report"] = self.bufs[8].clone()
            self.seen["flags"] = int(self.bufs[9][0])
            self.bufs[6][:] = torch.arange(NP, dtype=torch.float64) * (r + 1)
        elif k == 3:
            self.seen["grad"] = self.bufs[6].clone()
        elif k == 4:
            self._own(self.bufs[2], 2.0)
        elif k == 5:
            self.bufs[10].fill_(1.0 + r)
            self.bufs[11].fill_(1.0)


def _worker(rank, world, port, q, slab):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = FakeTrainer(rank, world, slab)
        f = PartitionedFrame(tr, TorchComm())
        f.step(2)
        img, sos = f.finish()
        q.put((rank, tr.log, {k: (v.numpy() if torch.is_tensor(v) else v) for k, v in tr.seen.items()},
               img.numpy(), sos.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("slab", [False, True])
def test_partitioned_frame_collectives_gloo(slab):
    world, port = 2, 29517 + int(slab)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, slab)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = H * W // world
    for rank, log, seen, img, sos in out:
        assert log == [0, 6, 7, 2, 3, 0, 6, 7, 2, 3, 4, 5]
        dv = np.zeros(H * W)
        if slab:
            dv[:n], dv[n:] = 1.0, 2.0  # each rank's slab, gathered
        else:
            dv = dv.reshape(H, W)
            dv[0::2], dv[1::2] = 1.0, 2.0  # each rank's rows, summed
        np.testing.assert_array_equal(seen["dv"].reshape(-1), dv.reshape(-1))
        gv = seen["gv"].reshape(-1)
        if slab:  # reduce-scatter: the owner's slab holds the sum
            np.testing.assert_array_equal(gv[rank * n:(rank + 1) * n], np.full(n, 0.5 + 1.0))
        else:
            np.testing.assert_array_equal(gv, np.full(H * W, 0.5 + 1.0))
        np.testing.assert_array_equal(seen["report"], np.array([1.0, 2.0, 3.0]) * 3)
        assert seen["flags"] == 4  # MAX
        np.testing.assert_array_equal(seen["grad"], np.arange(NP) * 3.0)
        np.testing.assert_allclose(img, np.full((H, W), 3.0 / 2.0))  # (1 + 2) / (1 + 1)
        np.testing.assert_allclose(sos, np.full((H, W), 1502.0))
