"""NTD apply time (slot-layout sweep alone, CUDA events, median) for a
BASELINE grid at a batch size: python tools/ntd_time.py cfg systems [ctas]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

if os.environ.get("VARIANT_LIB"):
    _lib.LIB_PATH = os.environ["VARIANT_LIB"]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nx, ny, nz = problems.CONFIGS[cfg]["grid"]
n = nx * ny * nz
kap = np.stack([problems.baseline_kappa(cfg, s % 4)[0] for s in range(S)])
a = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, problems.baseline_kappa(cfg, 0)[1])
pre, st = D.ntd_factor(a, nx, ny, nz, S)
solve = D.solve_bands(pre, nx, ny, nz, S)
work = torch.zeros(_lib.load().ntd_apply_work_doubles(nx, ny, nz, S), dtype=torch.float64, device="cuda")
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else D.ntd_ctas(S)
R = 10 if n * S < 3e7 else 3
fn = lambda: _lib.call("ntd_apply_slot_ex", _lib.ptr(solve), _lib.ptr(work), nx, ny, nz, S, None, ctas,  # noqa: E731
                       _lib.stream())
fn()
torch.cuda.synchronize()
ts = []
for _ in range(R):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    fn()
    e[1].record()
    torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]))
t = float(np.median(ts))
steps = (nz + 1) * (ny + 1)
print(f"cfg{cfg} {nx}x{ny}x{nz} systems {S} ctas {ctas}: {t:.3f} ms per apply, "
      f"{t * 1e-3 / steps * 1.965e9:.0f} cycles per line step (at 1965 MHz)", flush=True)
