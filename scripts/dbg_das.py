import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_util as gu  # noqa: E402
from oracle_lib import rel_l2  # noqa: E402
from paper_2409_10876_b200.api import Context  # noqa: E402

ctx = Context(0)
for name in ["das_edge", "das_cfg1_crop"]:
    z = gu.load(name)
    s = torch.as_tensor(z["sig"].astype(np.float32)).cuda()
    out = ctx.das_stack(s, gu.ring(z["ring"]), gu.meta(z["meta"]), gu.grid(z["grid"]),
                        float(z["v0"]), list(z["delays"]))
    got = out.double().cpu().numpy()
    want = z["out"]
    print(name, rel_l2(got, want))
    err = np.abs(got - want)
    for j in range(got.shape[0]):
        e = err[j]
        iy, ix = np.unravel_index(np.argmax(e), e.shape)
        print(" j", j, "rel", rel_l2(got[j], want[j]), "max at", (ix, iy), got[j, iy, ix],
              want[j, iy, ix])
