"""Break one cfg3 joint_reconstruct-equivalent frame into phases (wall + events)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2409_10876_b200 import workloads as wl
from paper_2409_10876_b200.api import Context, Trainer, joint_reconstruct

w = wl.cfg3()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, epochs=10, steps_per_epoch=1))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    tr.step(1); torch.cuda.synchronize(); t2 = time.perf_counter()
    tr.step(1); torch.cuda.synchronize(); t3 = time.perf_counter()
    tr.step(8); torch.cuda.synchronize(); t4 = time.perf_counter()
    out = tr.finish(); torch.cuda.synchronize(); t5 = time.perf_counter()
    tr.close(); torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"rep{rep}: create {1e3*(t1-t0):.1f} ms, step1 {1e3*(t2-t1):.1f}, step2 {1e3*(t3-t2):.1f}, "
          f"8 steps {1e3*(t4-t3):.1f}, finish {1e3*(t5-t4):.1f}, close {1e3*(t6-t5):.1f}")
for rep in range(3):
    t0 = time.perf_counter()
    joint_reconstruct(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, epochs=10, steps_per_epoch=1))
    torch.cuda.synchronize()
    print(f"joint_reconstruct {1e3*(time.perf_counter()-t0):.1f} ms")

# the bench's e2e call: 8 frames through joint_reconstruct_batch (traced)
from paper_2409_10876_b200.api import joint_reconstruct_batch  # noqa: E402
sigs = [wl.simulate(ctx, w, seed=f) for f in range(8)]
cfgs = [wl.train_config(w, epochs=10, steps_per_epoch=1, seed=f) for f in range(8)]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    joint_reconstruct_batch(ctx, sigs, w.ring, w.meta, w.grid, w.mask, cfgs)
    torch.cuda.synchronize()
    print(f"batch of 8: {1e3*(time.perf_counter()-t0):.1f} ms")
