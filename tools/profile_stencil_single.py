"""spmv+dot and true-residual kernels on one BASELINE system (for ncu): python tools/profile_stencil_single.py cfg"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nx, ny, nz = problems.CONFIGS[cfg]["grid"]
n = nx * ny * nz
kap, bc, _ = problems.baseline_kappa(cfg, 0)
a = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, bc)
a4 = D.sym_pack(a, nx, ny, nz, 1)
r = torch.rand((1, n), dtype=torch.float64, device="cuda")
cg = D.PcgDevice(a, nx, ny, nz, 1, 4, a4=a4)
cg.init(r, 1e-30)
cg.p.copy_(r)
cg.state[:, _lib.NTD_ST["RZ"]] = 1.0
for _ in range(3):
    _lib.call("ntd_pcg_spmv_alpha_sym", _lib.ptr(a4), _lib.ptr(cg.p), _lib.ptr(cg.ap), _lib.ptr(cg.state),
              _lib.ptr(cg.flags), _lib.ptr(cg.active), nx, ny, nz, 1, _lib.ptr(cg.work), _lib.stream())
    _lib.call("ntd_pcg_update_residual_sym", _lib.ptr(a4), _lib.ptr(r), _lib.ptr(cg.x), _lib.ptr(cg.r),
              _lib.ptr(cg.p), _lib.ptr(cg.ap), _lib.ptr(cg.state), _lib.ptr(cg.flags), _lib.ptr(cg.active),
              _lib.ptr(cg.history), 4, nx, ny, nz, 1, _lib.ptr(cg.work), _lib.stream())
torch.cuda.synchronize()
print("ok")
