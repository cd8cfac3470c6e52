"""Run the cfg3 step twice (fresh engines) and report per-parameter-block
bitwise agreement of the gradient (determinism triage).  Experiment driver."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2409_10876_b200 import workloads as wl  # noqa: E402
from paper_2409_10876_b200.api import Context, Trainer  # noqa: E402

w = wl.CONFIGS["cfg3"]()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
cfg = wl.train_config(w, seed=0, epochs=1, steps_per_epoch=int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                      use_cuda_graph=len(sys.argv) > 2)
gs = []
for _ in range(3):
    tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, cfg)
    tr.step(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
    gs.append(tr.read(6, (tr.n_params,), np.float64))
    tr.close()
H = 128
offs = [0, 3 * H]
for l in range(1, 4):
    offs.append(offs[-1] + H * H + H)
offs.append(offs[-1] + H + 1)
names = ["layer0", "layer1", "layer2", "layer3", "head"]
for k in (1, 2):
    for nm, a, b in zip(names, offs[:-1], offs[1:]):
        x, y = gs[0][a:b], gs[k][a:b]
        d = np.abs(x - y)
        print(f"run{k} {nm}: equal {np.array_equal(x, y)} n_diff {int((d > 0).sum())} max rel {d.max() / max(np.abs(x).max(), 1e-300):.2e}")
ctx.close()
