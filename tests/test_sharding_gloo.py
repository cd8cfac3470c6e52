"""CPU, world_size 2 over gloo: the cfg4 frame sharding used by bench.py is a
disjoint cover of the 8 frames, and the timing reduction is the max over ranks."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_10876_b200.workloads import shard_frames


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_frames(8, rank, world)
    lists = [None] * world
    dist.all_gather_object(lists, mine)
    t = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((lists, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_frame_sharding_and_max_timing_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    lists, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    flat = sorted(f for l in lists for f in l)
    assert flat == list(range(8))
    assert set(lists[0]).isdisjoint(lists[1])
    assert tmax == 11.0


def test_shard_frames_all_world_sizes():
    for world in (1, 2, 4, 8):
        got = sorted(f for r in range(world) for f in shard_frames(8, r, world))
        assert got == list(range(8))
        assert all(len(shard_frames(8, r, world)) == 8 // world for r in range(world))
