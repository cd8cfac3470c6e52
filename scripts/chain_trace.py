"""Timeline of CTA 0 of the fused SIREN forward (experiment build CHAIN_EXP=2).
PACT_LIB=build/rx/lib_c2.so python scripts/chain_trace.py"""
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
L.pact_debug_chain_trace.argtypes = [C.c_void_p, C.c_int]
w = wl.cfg3()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, use_cuda_graph=False))
tr.step(1)
torch.cuda.synchronize()
L.pact_debug_chain_trace(None, 1)
tr.phase(0)
torch.cuda.synchronize()
buf = np.zeros(3 * 1024 * 3, np.uint64)
L.pact_debug_chain_trace(buf.ctypes.data, 1)
ev = buf.reshape(3, 1024, 3).astype(np.int64)
names = {1: "mma layer start", 2: "mma ardy ok", 3: "mma wfull ok", 4: "mma layer issued",
         10: "epi tile start", 11: "epi first done", 12: "epi dfull ok", 13: "epi dfree", 14: "epi a_ready", 15: "epi head done"}
rows = []
for role in range(3):
    for tag, idx, t in ev[role]:
        if t > 0:
            rows.append((t, role, names.get(int(tag), str(tag)), int(idx)))
rows.sort()
t0 = rows[0][0]
for t, role, nm, i in rows[:140]:
    print(f"{(t - t0) / 1e3:9.3f} us  role{role}  {nm:18s} {i}")
