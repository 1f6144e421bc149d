"""Launch the stencil / CG kernels on a config-4 batch for ncu (profiling aid).
    python tools/profile_stencil.py [systems]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ins = [problems.baseline_config(4, s % 8) for s in range(min(B, 8))]
nx, ny, nz = ins[0][2]
n = nx * ny * nz
a = torch.from_numpy(np.stack([ins[s % len(ins)][0] for s in range(B)])).cuda()
a4 = D.sym_pack(a, nx, ny, nz, B)
r, w = torch.rand((B, n), dtype=torch.float64, device="cuda"), torch.rand((B, n), dtype=torch.float64, device="cuda")
t = torch.empty_like(r)
cg = D.PcgDevice(a, nx, ny, nz, B, 2, a4=a4)
cg.init(r, 1e-30)
cg.p.copy_(w)
for _ in range(2):
    D.residual(a, r, w, nx, ny, nz, B, t=t, a4=a4)
    cg.step_update()
torch.cuda.synchronize()
print("ok")
