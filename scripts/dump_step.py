"""One cfg3 iteration; saves dL/dv (buffer 5) and grad theta (6) to an .npz, for
A/B comparisons of kernel variants selected by environment switches.

    python scripts/dump_step.py out.npz [--cfg cfg3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_10876_b200 import workloads as wl  # noqa: E402
from paper_2409_10876_b200.api import Context, Trainer, make_patch_layout  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--cfg", default="cfg3")
args = ap.parse_args()
w = wl.CONFIGS[args.cfg]()
ctx = Context(0)
sig = wl.simulate(ctx, w, seed=0)
tr = Trainer(ctx, sig, w.ring, w.meta, w.grid, w.mask, wl.train_config(w, use_cuda_graph=False))
tr.step(1)
H, W = w.grid.height, w.grid.width
n_rays = w.n_angles * make_patch_layout(w.grid, w.patch_mm, w.overlap).n_patches
np.savez(args.out, gv=tr.read(5, (H, W), np.float64), grad=tr.read(6, (tr.n_params,), np.float64),
         w=tr.read(3, (n_rays,), np.float32), dw=tr.read(4, (n_rays,), np.float32))
tr.close()
ctx.close()
