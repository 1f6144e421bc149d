"""Per-warp cycle split of the hyperplane ILU0 kernel (CTA 0, variant build
with -DHP_TIMING): VARIANT_LIB=build/var/libntdgpu_hpt.so python tools/hp_timing.py cfg [nc w]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

_lib.LIB_PATH = os.environ["VARIANT_LIB"]
cfg = int(sys.argv[1])
nx, ny, nz = problems.CONFIGS[cfg]["grid"]
n = nx * ny * nz
kap = problems.baseline_kappa(cfg, 0)[0][None]
a = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, problems.baseline_kappa(cfg, 0)[1])
split = n // 2
f, _ = D.ilu0_factor(a, nx, ny, nz, 1, split)
skew = D.ilu0_skew_build(f, split, nx, ny, nz, 1)
work = torch.empty(_lib.load().ntd_ilu0_skew_work_doubles(nx, ny, nz, 1), dtype=torch.float64, device="cuda")
v = torch.rand((1, n), dtype=torch.float64, device="cuda")
z = torch.empty_like(v)
hp = (int(sys.argv[2]), int(sys.argv[3])) + ((int(sys.argv[4]),) if len(sys.argv) > 4 else ()) if len(sys.argv) > 3 else D.ilu0_hp_config(nx, ny, nz, split, 1)
lib = _lib.load()
lib.ntd_hp_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 128)()
D.ilu0_apply(f, split, v, nx, ny, nz, 1, z=z, skew=skew, work=work, hp=hp)
lib.ntd_hp_timing(buf, 1)
D.ilu0_apply(f, split, v, nx, ny, nz, 1, z=z, skew=skew, work=work, hp=hp)
lib.ntd_hp_timing(buf, 0)
t = np.array(buf[:]).reshape(32, 4)
print(f"cfg{cfg} hp {hp}: per warp (CTA 0, fwd+bwd): work / barrier cycles per step")
for w in range(hp[1]):
    st = max(1, t[w, 3])
    print(f"  warp {w:2d}: steps {t[w, 3]}, work {t[w, 0] / st:7.0f}, barrier {t[w, 2] / st:7.0f}")
