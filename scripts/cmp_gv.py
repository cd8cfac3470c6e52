import sys
import numpy as np
a, b = np.load(sys.argv[1])["gv"], np.load(sys.argv[2])["gv"]
d = np.abs(a - b)
scale = np.abs(b).max()
print("max |b|", scale, "max diff", d.max(), "at", np.unravel_index(d.argmax(), d.shape))
big = d > 1e-6 * scale
print("pixels with diff > 1e-6 max:", big.sum(), "of", big.size)
ys, xs = np.nonzero(big)
if len(ys):
    print("rows", np.unique(ys)[:20], "cols", np.unique(xs)[:20])
    print("border share", np.mean((ys == 0) | (xs == 0) | (ys == a.shape[0]-1) | (xs == a.shape[1]-1)))
inner = slice(1, -1)
print("interior rel L2", np.linalg.norm((a-b)[inner, inner]) / np.linalg.norm(b[inner, inner]))
print("border rel L2", np.linalg.norm(np.concatenate([(a-b)[0], (a-b)[-1], (a-b)[:, 0], (a-b)[:, -1]])) /
      np.linalg.norm(np.concatenate([b[0], b[-1], b[:, 0], b[:, -1]])))
