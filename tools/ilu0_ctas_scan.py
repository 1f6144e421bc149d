"""ILU0 skew apply time vs CTAs per system half (cluster size), config-4 systems.
    python tools/ilu0_ctas_scan.py [B1,B2,...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402
from paper_1909_09771_b200.batch import BatchSolver  # noqa: E402

sizes = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,8").split(",")]
ins = [problems.baseline_config(4, s) for s in range(max(sizes))]
nx, ny, nz = ins[0][2]
for B in sizes:
    a = torch.from_numpy(np.stack([i[0] for i in ins[:B]])).cuda()
    s = BatchSolver(a, nx, ny, nz, groups=1).setup()
    P = s.precond
    v = torch.rand((B, nx * ny * nz), dtype=torch.float64, device="cuda")
    x = torch.empty_like(v)
    row = []
    for c in ((1, 24), (2, 24), (4, 24), (2, 12), (4, 12), (4, 8), (8, 6), (8, 8), (4, 6), (8, 12)):
        D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, B, z=x, skew=P.skew, ctas=c)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(5):
            D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, B, z=x, skew=P.skew, ctas=c)
        e[1].record()
        torch.cuda.synchronize()
        row.append(f"{c[0]}x{c[1]}:{e[0].elapsed_time(e[1]) / 5:.3f}")
    print(f"B={B} ms by ctas/half:", " ".join(row), flush=True)
