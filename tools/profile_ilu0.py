"""Run the ILU0 apply a few times for ncu (python tools/profile_ilu0.py cfg systems [hp|skew])."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

cfg = int(sys.argv[1])
S = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "hp"
nx, ny, nz = problems.CONFIGS[cfg]["grid"]
n = nx * ny * nz
kap = np.stack([problems.baseline_kappa(cfg, s % 4)[0] for s in range(S)])
a = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, problems.baseline_kappa(cfg, 0)[1])
split = n // 2
f, _ = D.ilu0_factor(a, nx, ny, nz, S, split)
skew = D.ilu0_skew_build(f, split, nx, ny, nz, S)
work = torch.empty(_lib.load().ntd_ilu0_skew_work_doubles(nx, ny, nz, S), dtype=torch.float64, device="cuda")
v = torch.rand((S, n), dtype=torch.float64, device="cuda")
z = torch.empty_like(v)
hp = D.ilu0_hp_config(nx, ny, nz, split, S) if mode == "hp" else None
for _ in range(3):
    D.ilu0_apply(f, split, v, nx, ny, nz, S, z=z, skew=skew, work=work, hp=hp)
torch.cuda.synchronize()
print("done", hp)
