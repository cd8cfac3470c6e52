"""Per-block errors of the width-256 SIREN vs the oracle (debug helper)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from oracle_lib import orc, rel_l2
from paper_2409_10876_b200.api import CircularMask, GridSpec, SirenSpec, init_siren, masked_pixels, Context
ctx = Context(0)
for (width, height, layers, seed) in [(97, 83, 4, 13), (64, 64, 2, 5)]:
    grid = GridSpec(width, height, 1e-4, -0.5e-4 * width, -0.5e-4 * height)
    mask = CircularMask(0.0, 0.0, 0.45e-4 * max(width, height))
    spec = SirenSpec(256, layers, 30.0, 100.0, 1500.0)
    theta = init_siren(seed, spec)
    rng = np.random.default_rng(seed)
    theta = theta * (1.0 + 0.05 * rng.standard_normal(theta.shape))
    _, dev = ctx.render_sos(spec, torch.as_tensor(theta), grid, mask)
    want = orc().render_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask)
    print("case", width, height, layers, "render", rel_l2(dev.double().cpu().numpy(), want - spec.v0))
    idx, _ = masked_pixels(grid, mask)
    g = np.random.default_rng(100 + seed).standard_normal(len(idx)).astype(np.float32)
    got = ctx.siren_backward(spec, torch.as_tensor(theta), grid, mask, torch.as_tensor(g)).cpu().numpy()
    want = orc().backprop_sos(spec, theta.astype(np.float32).astype(np.float64), grid, mask, g.astype(np.float64))
    off = 0
    for l in range(layers + 1):
        rows = 1 if l == layers else 256
        cols = 2 if l == 0 else 256
        W = slice(off, off + rows * cols); B = slice(off + rows * cols, off + rows * cols + rows)
        print(f"  layer {l}: W {rel_l2(got[W], want[W]):.3e} b {rel_l2(got[B], want[B]):.3e}")
        off += rows * cols + rows
