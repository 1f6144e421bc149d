"""Where the ILU0 skew sweep spends its time (debug build with -DSKEW_TIMING):
    NTD_LIB_OVERRIDE=build/var/libntdgpu_skt.so python tools/skew_timing.py [systems]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402
from paper_1909_09771_b200.batch import BatchSolver  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ins = [problems.baseline_config(4, s) for s in range(B)]
nx, ny, nz = ins[0][2]
a = torch.from_numpy(np.stack([i[0] for i in ins])).cuda()
s = BatchSolver(a, nx, ny, nz, groups=1).setup()
P = s.precond
v = torch.rand((B, nx * ny * nz), dtype=torch.float64, device="cuda")
x = torch.empty_like(v)
lib = _lib.load()
fn = lib.ntd_skew_timing
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 4)()
env = os.environ.get("SKEW_CTAS")  # "c,w"
ctas = tuple(int(t) for t in env.split(",")) if env else P.ilu_ctas
D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, B, z=x, skew=P.skew, ctas=ctas)
torch.cuda.synchronize()
fn(buf, 1)
R = 5
for _ in range(R):
    D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, B, z=x, skew=P.skew, ctas=ctas)
torch.cuda.synchronize()
fn(buf, 1)
wait, total, steps, units = (buf[i] / R for i in range(4))
print(f"block 0, per apply (fwd+bwd), summed over its warps: total {total:.0f} cyc, waiting {wait:.0f} "
      f"({100 * wait / total:.1f}%), steps {steps:.0f}, units {units:.0f}; "
      f"per warp-step {total / steps:.0f} cyc, of which waiting {wait / steps:.0f}")
