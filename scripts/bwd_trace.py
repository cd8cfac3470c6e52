"""Timeline of one CTA of the middle-layer SIREN backward kernel (a library built
with -DBWD_EXP=5: globaltimer stamps per role and tile).  Experiment driver.

    PACT_LIB=build/trace/libpact_cuda.so python scripts/bwd_trace.py
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2409_10876_b200 import _abi  # noqa: E402
from paper_2409_10876_b200 import workloads as wl  # noqa: E402
from paper_2409_10876_b200.api import Context, Trainer  # noqa: E402

w = wl.CONFIGS["cfg3"]()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, use_cuda_graph=False))
tr.step(2)
torch.cuda.synchronize()
lib = _abi.lib()
fn = lib.pact_debug_bwd_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((16, 512), dtype=np.uint64)
fn(None, 1)
tr.step(1)
torch.cuda.synchronize()
fn(buf.ctypes.data, 0)
t0 = buf[buf > 0].min()
F16 = os.environ.get("BWD16", "1") == "1"
if F16:  # siren_bwd16.cu tags
    names = {1: "dA xfull", 12: "dA read", 14: "dA split", 13: "dA pfree", 2: "dA gready", 5: "z rfull",
             6: "z zfree", 7: "z zready", 8: "mma w-issue", 9: "mma g-issue", 10: "epi dfull"}
else:
    names = {1: "dA xfull", 12: "dA hi-ld", 14: "dA comp", 3: "dA tfree", 4: "dA tready", 13: "dA lo-st",
             2: "dA gready", 5: "z rfull", 6: "z wfree", 11: "z stored", 7: "z zready", 8: "mma w-issue",
             9: "mma g-issue", 10: "epi dfull"}
ntile = int((buf[1] > 0).sum())
print("tiles", ntile)
rel = np.where(buf > 0, (buf.astype(np.int64) - int(t0)), -1)
order = [1, 12, 14, 13, 2, 5, 6, 7, 8, 9, 10] if F16 else [1, 12, 14, 3, 4, 13, 2, 5, 6, 11, 7, 8, 9, 10]
print("tile " + " ".join(f"{names[t]:>11s}" for t in order))
for i in list(range(0, 8)) + list(range(20, 26)) + list(range(ntile - 3, ntile)):
    print(f"{i:4d} " + " ".join(f"{rel[t, i]:11d}" for t in order))
# steady-state per-tile period and mean gaps
lo, hi = 10, ntile - 5
per = (rel[1, hi] - rel[1, lo]) / (hi - lo)
print("period ns/tile", per)
pairs = ([(1, 12), (12, 14), (14, 13), (13, 2), (5, 6), (6, 7), (2, 8), (7, 8), (8, 9), (9, 10)] if F16 else
         [(1, 12), (12, 14), (14, 3), (3, 4), (4, 13), (13, 2), (5, 6), (6, 11), (11, 7), (4, 8), (7, 8), (8, 9), (9, 10)])
for a, b in pairs:
    print(f"{names[a]:>11s} -> {names[b]:>11s}: {np.mean(rel[b, lo:hi] - rel[a, lo:hi]):8.1f} ns")
# cross-tile gaps
print("gready(i-1) -> xfull(i):", np.mean(rel[1, lo + 1:hi] - rel[2, lo:hi - 1]))
print("zready(i-1) -> rfull(i):", np.mean(rel[5, lo + 1:hi] - rel[7, lo:hi - 1]))
print("g-issue(i-1) -> w-issue(i):", np.mean(rel[8, lo + 1:hi] - rel[9, lo:hi - 1]))
print("dfull(i-1) -> dfull(i):", np.mean(rel[10, lo + 1:hi] - rel[10, lo:hi - 1]))
tr.close()
ctx.close()
