"""Launch the hot kernels on a config-4 sub-batch for ncu (debug/profiling aid).

    PROFILE_BATCH=64 python tools/profile_kernels.py [systems]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402
from paper_1909_09771_b200.batch import BatchSolver  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ins = [problems.baseline_config(4, s) for s in range(B)]
nx, ny, nz = ins[0][2]
a = torch.from_numpy(np.stack([i[0] for i in ins])).cuda()
xt = torch.from_numpy(np.stack([i[1] for i in ins])).cuda()
b = torch.empty_like(xt)
_lib.call("ntd_spmv", _lib.ptr(a), _lib.ptr(xt), _lib.ptr(b), nx, ny, nz, B, None, _lib.stream())
s = BatchSolver(a, nx, ny, nz, groups=1).setup()
v = torch.rand_like(b)
x = torch.empty_like(b)
P = s.precond
# the CTA mappings the solver uses for the whole batch it belongs to
# (PROFILE_BATCH systems on the GPU; bench.py: 64 in 16 stream groups)
full = int(os.environ.get("PROFILE_BATCH", "64"))
ilu_ctas, ntd_ctas = D.ilu0_ctas(full), D.ntd_ctas(full)
for _ in range(2):
    # the NTD sweep as the solver launches it (slot layout, ctas per system)
    _lib.call("ntd_apply_slot_ex", _lib.ptr(P.solve), _lib.ptr(P.work), nx, ny, nz, B, None, ntd_ctas,
              _lib.stream())
    D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, B, z=x, skew=P.skew, ctas=ilu_ctas,
                 hp=D.ilu0_hp_config(nx, ny, nz, P.split, full))
    D.residual(a, v, x, nx, ny, nz, B, a4=s.precond.a4)
torch.cuda.synchronize()
print("ok")
