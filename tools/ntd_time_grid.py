"""NTD apply time on an arbitrary grid (lane-layout sweep alone, CUDA events, median):
python tools/ntd_time_grid.py nx ny nz [systems]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

if os.environ.get("VARIANT_LIB"):
    _lib.LIB_PATH = os.environ["VARIANT_LIB"]
nx, ny, nz = (int(v) for v in sys.argv[1:4])
S = int(sys.argv[4]) if len(sys.argv) > 4 else 1
rng = np.random.default_rng(1)
kap = np.exp(rng.normal(0.0, 1.0, (S, nz, ny, nx)))
a = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, (True,) * 6)
pre, st = D.ntd_factor(a, nx, ny, nz, S)
solve = D.solve_bands(pre, nx, ny, nz, S)
work = torch.zeros(_lib.load().ntd_apply_work_doubles(nx, ny, nz, S), dtype=torch.float64, device="cuda")
fn = lambda: _lib.call("ntd_apply_slot_ex", _lib.ptr(solve), _lib.ptr(work), nx, ny, nz, S, None, 2,  # noqa: E731
                       _lib.stream())
fn()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    fn()
    e[1].record()
    torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]))
t = float(np.median(ts))
steps = (nz + 1) * (ny + 1)
print(f"{nx}x{ny}x{nz} systems {S}: {t:.3f} ms per apply, {t * 1e-3 / steps * 1.965e9:.0f} cycles per line step "
      f"(at 1965 MHz)", flush=True)
