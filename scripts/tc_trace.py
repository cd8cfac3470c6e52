"""Timeline of CTA 0 of one forward tcgen05 layer (experiment build TC_EXP=5).
PACT_LIB=build/exp/libpact_exp5.so python scripts/tc_trace.py"""
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
L.pact_debug_trace.argtypes = [C.c_void_p, C.c_int, C.c_int]
w = wl.cfg3()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, use_cuda_graph=False))
tr.step(1)
torch.cuda.synchronize()
L.pact_debug_trace(None, 0, 1)  # reset
tr.phase(0)  # the forward: 3 tc layers, trace keeps the first 4096 events
torch.cuda.synchronize()
buf = np.zeros(3 * 4096, np.uint64)
n = L.pact_debug_trace(buf.ctypes.data, 4096, 1)
ev = buf[: 3 * n].reshape(-1, 3).astype(np.int64)
ev = ev[ev[:, 2] > 0]
t0 = ev[:, 2].min()
names = {1: "raw_wait_start", 2: "raw_ready", 3: "buf_free", 4: "transform_done", 5: "issue_start",
         6: "epi_wait", 7: "epi_full", 8: "epi_done"}
# first kernel only: stop when a tile index restarts after an epi_done
rows = []
for tag, idx, t in ev:
    rows.append((t - t0, names[int(tag)], int(idx)))
rows.sort()
for t, nm, i in rows[:160]:
    print(f"{t/1000:9.2f} us  {nm:16s} {i}")
