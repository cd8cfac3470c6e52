"""Timeline of CTA 0 of the middle-layer fused SIREN backward (BWD_EXP=5 build).
PACT_LIB=/tmp/bx/lib5.so python scripts/bwd_trace.py"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2409_10876_b200 import _abi  # noqa: E402
from paper_2409_10876_b200 import workloads as wl  # noqa: E402
from paper_2409_10876_b200.api import Context, Trainer  # noqa: E402

L = _abi.lib()
L.pact_debug_bwd_trace.argtypes = [C.c_void_p, C.c_int]
w = wl.cfg3()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, use_cuda_graph=False))
tr.step(1)
tr.phase(0)
tr.phase(1)
torch.cuda.synchronize()
L.pact_debug_bwd_trace(None, 1)
tr.phase(2)
torch.cuda.synchronize()
buf = np.zeros(16 * 512, np.uint64)
L.pact_debug_bwd_trace(buf.ctypes.data, 1)
ev = buf.reshape(16, 512).astype(np.int64)
names = {1: "D start", 2: "D gfree", 3: "D tfree", 4: "D tready>", 5: "Z rfull", 6: "Z wfree",
         7: "Z zready>", 8: "M w-ready", 9: "M g-ready", 10: "E dfull", 11: "Z stored", 12: "D loaded",
         13: "D stored", 14: "D computed"}
K = sorted(names)
t0 = ev[ev > 0].min()
n = int((ev[1] > 0).sum())
print("tiles", n, "span us", (ev[ev > 0].max() - t0) / 1e3)
print("tile " + " ".join(f"{names[k]:>9s}" for k in K))
for i in list(range(0, 8)) + list(range(n - 4, n)):
    print(f"{i:4d} " + " ".join(f"{(ev[k, i] - t0) / 1e3 if ev[k, i] else float('nan'):9.2f}" for k in K))
d = np.diff(ev[8, :n]) / 1e3
print("mean tile period (M wready) us", d[4:].mean())
