"""Small solves for a quick end-to-end check (compute-sanitizer is not available on this pool):
    python tools/sanitize_small.py [wide]
Grids cover K = 1, 2 (PIPE ring mode), degenerate ny / nz, odd sizes; one wide grid (K = 6) covers the
non-pipelined mode."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_09771_b200 as ntd  # noqa: E402
from paper_1909_09771_b200 import problems  # noqa: E402

rng = np.random.default_rng(0)
grids = [(7, 5, 4), (33, 3, 2), (40, 9, 6), (16, 1, 3), (5, 6, 1), (12, 12, 12)]
if len(sys.argv) > 1 and sys.argv[1] == "wide":
    grids = [(170, 6, 5)]
for (nx, ny, nz) in grids:
    kap = 10.0 ** rng.uniform(-1, 1, (nz, ny, nx))
    data = problems.assemble_kappa(kap, nx, ny, nz)
    a = ntd.BandedMatrix(nx, ny, nz, data)
    pre = ntd.factor_level3(a)
    v = rng.uniform(-1, 1, a.n_rows)
    x = ntd.ntd_apply(pre, v)
    cp = ntd.CombinedPrecond(a)
    b = ntd.spmv(a, v)
    xs, st = ntd.pcg(a, b, cp, tol=1e-8)
    print(nx, ny, nz, "iterations", st.iterations, "err", float(np.abs(xs - v).max()), flush=True)
torch.cuda.synchronize()
print("ok")
