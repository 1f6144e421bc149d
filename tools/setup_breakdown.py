"""Setup-time breakdown of CombinedPrecond on one BASELINE system (CUDA events around each setup step)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import problems  # noqa: E402
from paper_1909_09771_b200 import _lib  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

if os.environ.get("VARIANT_LIB"):
    _lib.LIB_PATH = os.environ["VARIANT_LIB"]

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nx, ny, nz = problems.CONFIGS[cfg]["grid"]
n = nx * ny * nz
kap, bc, _ = problems.baseline_kappa(cfg, 0)
a = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, bc)
torch.cuda.synchronize()
steps = [
    ("ntd_factor", lambda: D.ntd_factor(a, nx, ny, nz, 1)),
    ("ilu0_factor", lambda: D.ilu0_factor(a, nx, ny, nz, 1, n // 2)),
    ("check_grid_pattern", lambda: D.check_grid_pattern(a, nx, ny, nz)),
    ("sym_pack", lambda: D.sym_pack(a, nx, ny, nz, 1)),
]
for rep in range(2):
    res = {}
    for name, fn in steps:
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        out = fn()
        e[1].record()
        torch.cuda.synchronize()
        res[name] = e[0].elapsed_time(e[1])
        if name == "ntd_factor":
            pre = out[0]
        if name == "ilu0_factor":
            f = out[0]
    for name, fn in (("solve_bands", lambda: D.solve_bands(pre, nx, ny, nz, 1)),
                     ("ilu0_skew_build", lambda: D.ilu0_skew_build(f, n // 2, nx, ny, nz, 1))):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        fn()
        e[1].record()
        torch.cuda.synchronize()
        res[name] = e[0].elapsed_time(e[1])
print(f"cfg{cfg} setup ms:", {k: round(v, 1) for k, v in res.items()}, "total", round(sum(res.values()), 1))
