"""Where does the NTD apply differ from the oracle on a BASELINE config?
    python tools/parity_probe.py CFG
Splits the end-to-end apply error into the factor part and the apply part."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402
import paper_1909_09771_b200 as ntd  # noqa: E402
from paper_1909_09771_b200 import problems  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def rel2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
data, xt, (nx, ny, nz) = problems.baseline_config(cfg)
a = ntd.BandedMatrix(nx, ny, nz, data)
pre = ntd.factor_level3(a)
pre_o = oracle.factor_level3(data, nx, ny, nz, nthreads=2)
pg = pre.host()
print("factor rel per band", [f"{rel(pg[i], pre_o[i]):.2e}" for i in range(7)])
print("factor bitwise-equal fraction per band", [f"{np.mean(pg[i] == pre_o[i]):.4f}" for i in range(7)])
v = np.random.default_rng(5).uniform(-1, 1, a.n_rows)
yo = oracle.ntd_apply(pre_o, v, nx, ny, nz, nthreads=2)
yg = ntd.ntd_apply(pre, v)
print(f"end-to-end apply: max-rel {rel(yg, yo):.3e}  2-rel {rel2(yg, yo):.3e}")
po = ntd.PreconBands(nx, ny, nz, bands=torch.from_numpy(pre_o).cuda())
yg_o = ntd.ntd_apply(po, v)
print(f"GPU apply on the oracle factor: max-rel {rel(yg_o, yo):.3e}  2-rel {rel2(yg_o, yo):.3e}")
yo_g = oracle.ntd_apply(np.ascontiguousarray(pg), v, nx, ny, nz, nthreads=2)
print(f"oracle apply on the GPU factor vs oracle/oracle: max-rel {rel(yo_g, yo):.3e}  2-rel {rel2(yo_g, yo):.3e}")
i = int(np.argmax(np.abs(yg - yo)))
print("worst index", i, "cell", (i % nx, (i // nx) % ny, i // (nx * ny)), yg[i], yo[i])
