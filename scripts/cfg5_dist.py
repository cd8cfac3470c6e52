"""cfg5 (one 2048^2 frame) over N GPUs: python -m torch.distributed.run --nnodes=1
--nproc-per-node N --master-addr 127.0.0.1 --master-port P scripts/cfg5_dist.py [--steps K]

Rank 0 simulates the signals and broadcasts them; every rank builds its
partition of the frame (pact_trainer_create_partitioned) and steps it with
distributed.PartitionedFrame (NCCL all-reduces between phases).  Prints one
JSON line on rank 0: ms per iteration (CUDA events on the engine streams, max
over ranks), the loss report and the final-image timing.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2409_10876_b200 import workloads as wl  # noqa: E402
from paper_2409_10876_b200.api import Context, Trainer  # noqa: E402
from paper_2409_10876_b200.distributed import PartitionedFrame, TorchComm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--cfg", default="cfg5")
args = ap.parse_args()

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
w = wl.CONFIGS[args.cfg]()
ctx = Context(local)
if rank == 0:
    sig = wl.simulate(ctx, w, seed=0)
else:
    sig = torch.empty((w.ring.n_transducers, w.meta.n_samples), device="cuda")
dist.broadcast(sig, 0)
torch.cuda.synchronize()
t0 = time.perf_counter()
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, use_cuda_graph=False),
             partition=(rank, world))
frame = PartitionedFrame(tr, TorchComm())
torch.cuda.synchronize()
create_s = time.perf_counter() - t0
frame.step(args.warmup)
dist.barrier()
torch.cuda.synchronize()
eng = tr.stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(eng)
frame.step(args.steps)
b.record(eng)
torch.cuda.synchronize()
t = torch.tensor([a.elapsed_time(b) / args.steps], device="cuda", dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
rep = tr.report(1)
a.record(eng)
img, sos = frame.finish()
b.record(eng)
torch.cuda.synchronize()
if rank == 0:
    print(json.dumps({"config": args.cfg, "world": world, "ms_per_iteration": float(t.item()),
                      "create_s": create_s, "finish_ms": a.elapsed_time(b), "report": rep,
                      "local": tr.local()}), flush=True)
tr.close()
ctx.close()
dist.destroy_process_group()
