"""One cfg3 frame: build the engine, run a few NF-APACT iterations eagerly
(no CUDA graph) so ncu sees each kernel launch.  Used for the profiles/ captures.

    python scripts/profile_iter.py [--steps 3] [--cfg cfg3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2409_10876_b200 import workloads as wl  # noqa: E402
from paper_2409_10876_b200.api import Context, Trainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--cfg", default="cfg3")
args = ap.parse_args()

w = wl.CONFIGS[args.cfg]()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask,
             wl.train_config(w, use_cuda_graph=False))
tr.step(args.steps)
print("report", tr.report(1))
for _ in range(2):
    print("stages", tr.profile_step())
torch.cuda.synchronize()
tr.close()
ctx.close()
