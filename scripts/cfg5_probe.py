"""One cfg5 frame on one GPU: simulate, trainer create, a few iterations, stage profile."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import Context, Trainer

w = wl.cfg5()
ctx = Context(0)
t0 = time.perf_counter()
sig = wl.simulate(ctx, w, seed=0)
torch.cuda.synchronize()
print("simulate s", time.perf_counter() - t0, tuple(sig.shape), flush=True)
t0 = time.perf_counter()
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, use_cuda_graph=False))
torch.cuda.synchronize()
print("create s", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter()
tr.step(1)
torch.cuda.synchronize()
print("first step s", time.perf_counter() - t0, flush=True)
print("report", tr.report(1))
print("stages", tr.profile_step())
print("mem GB", torch.cuda.max_memory_allocated() / 1e9)
tr.close()
ctx.close()
