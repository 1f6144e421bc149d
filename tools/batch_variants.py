"""Config-4 batch (64 x 96^3) solve rate under different ILU0 / NTD mapping
policies (experiments; the product picks them in device.ilu0_hp_config /
ilu0_ctas / ntd_ctas).  python tools/batch_variants.py policy [systems] [groups]
policies: auto, skew, hp:nc:w[:links] (fixed), hpmin (hp whenever it fits)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402
from paper_1909_09771_b200.batch import BatchSolver  # noqa: E402

if os.environ.get("VARIANT_LIB"):  # experiments: a variant build (tools/variant_lib.sh)
    _lib.LIB_PATH = os.environ["VARIANT_LIB"]
policy = sys.argv[1] if len(sys.argv) > 1 else "auto"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 64
GROUPS = int(sys.argv[3]) if len(sys.argv) > 3 else None
orig = D.ilu0_hp_config
if policy == "skew":
    D.ilu0_hp_config = lambda *a, **k: None
elif policy.startswith("hp:"):
    cfg_ = tuple(int(v) for v in policy.split(":")[1:])  # nc, w[, links]
    D.ilu0_hp_config = lambda *a, **k: cfg_
elif policy == "hpmin":
    D.ilu0_hp_config = lambda nx, ny, nz, split, systems: orig(nx, ny, nz, split, 1)
nx, ny, nz = problems.CONFIGS[4]["grid"]
n = nx * ny * nz
kaps, xts = [], []
for s in range(S):
    kap, bc, rng = problems.baseline_kappa(4, s)
    kaps.append(kap)
    xts.append(rng.uniform(-1.0, 1.0, n))
a = D.assemble(torch.from_numpy(np.stack(kaps)).cuda(), nx, ny, nz, bc)
xt = torch.from_numpy(np.stack(xts)).cuda()
b = torch.empty_like(xt)
_lib.call("ntd_spmv", _lib.ptr(a), _lib.ptr(xt), _lib.ptr(b), nx, ny, nz, S, None, _lib.stream())
solver = BatchSolver(a, nx, ny, nz, groups=GROUPS).setup()
solver.reserve(4)
solver.solve_many([b] * 2, 1e-8, x_outs=[solver.x] * 2)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
res = solver.solve_many([b] * 3, 1e-8, x_outs=[solver.x] * 3)
e[1].record()
torch.cuda.synchronize()
work = sum(n * sum(r.iterations) for r in res)
print(f"policy {policy} systems {S} groups {len(solver.groups)}: {work / (e[0].elapsed_time(e[1]) / 1e3) / 1e6:.0f} Munk-iter/s, "
      f"iters {min(res[0].iterations)}-{max(res[0].iterations)}", flush=True)
