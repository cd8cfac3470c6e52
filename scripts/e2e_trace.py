"""e2e call timing with host-side trainer-creation traces (PACT_TRACE=1)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import Context, joint_reconstruct_batch
w = wl.CONFIGS["cfg3"]()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
cfgs = [wl.train_config(w, epochs=10, steps_per_epoch=1, seed=f) for f in range(8)]
sigs = [sig.cpu().pin_memory() for _ in range(8)]
for rep in range(3):
    torch.cuda.synchronize(); t = time.time()
    joint_reconstruct_batch(ctx, sigs, w.ring, w.meta, w.grid, w.mask, cfgs)
    torch.cuda.synchronize(); print("call s", time.time() - t, file=sys.stderr)
