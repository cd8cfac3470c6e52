"""Relative L2 differences of matching arrays in two .npz files."""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    x, y = a[k].astype(np.float64), b[k].astype(np.float64)
    print(k, "rel L2 %.3e" % (np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)),
          "bitwise" if np.array_equal(a[k], b[k]) else "")
