"""ILU0 apply time (fwd + bwd, CUDA events, median of R) of the skewed
progress-word kernel vs the hyperplane kernel for several (CTAs per half,
warps) mappings, on the BASELINE grids at a given batch size.
python tools/ilu0_hp_scan.py [cfg] [systems]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402

if os.environ.get("VARIANT_LIB"):  # experiments: a variant build (tools/variant_lib.sh)
    _lib.LIB_PATH = os.environ["VARIANT_LIB"]
QUICK = os.environ.get("QUICK") == "1"  # only the auto hp mapping
LINKS = int(os.environ.get("LINKS", "0"))  # 1 cluster, 2 global-memory links, 0 the kernel's default

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nx, ny, nz = problems.CONFIGS[cfg]["grid"]
n = nx * ny * nz
kap = np.stack([problems.baseline_kappa(cfg, s)[0] for s in range(min(S, 4))])
kap = np.concatenate([kap] * (-(-S // kap.shape[0])))[:S]
bc = problems.baseline_kappa(cfg, 0)[1]
a = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, bc)
split = n // 2
f, st = D.ilu0_factor(a, nx, ny, nz, S, split)
skew = D.ilu0_skew_build(f, split, nx, ny, nz, S)
work = torch.empty(_lib.load().ntd_ilu0_skew_work_doubles(nx, ny, nz, S), dtype=torch.float64, device="cuda")
v = torch.rand((S, n), dtype=torch.float64, device="cuda")
z_ref = torch.empty_like(v)
D.ilu0_apply(f, split, v, nx, ny, nz, S, z=z_ref)
R = 10 if n * S < 5e7 else 3


def timed(fn):
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
    return float(np.median(ts))


auto = D.ilu0_hp_config(nx, ny, nz, split, S)
print(f"cfg{cfg} {nx}x{ny}x{nz} systems {S}: auto hp = {auto}", flush=True)
if QUICK and auto is not None:
    z = torch.empty_like(v)
    t = timed(lambda: D.ilu0_apply(f, split, v, nx, ny, nz, S, z=z, skew=skew, work=work, hp=auto))
    print(f"  hp {auto}: {t:.3f} ms  bitwise={torch.equal(z, z_ref)}", flush=True)
    sys.exit(0)
for ctas in ((1, 24), (2, 24), (4, 12), (8, 6)):
    z = torch.empty_like(v)
    t = timed(lambda: D.ilu0_apply(f, split, v, nx, ny, nz, S, z=z, skew=skew, work=work, ctas=ctas, hp=None))
    print(f"  skew {ctas}: {t:.3f} ms  bitwise={torch.equal(z, z_ref)}", flush=True)
g = (ny + 31) // 32
nk = nz - split // (nx * ny)
for nc in (1, 2, 4, 8, 16, 24, 37, 48, 74):
    if nc > nk or (nc > 16 and S > 1):
        continue
    umax = -(-nk // nc) * g
    for w in (4, 8, 12, 16, 24):
        upw = -(-umax // w)
        if upw > 8 or (w > 16 and upw > 1) or umax > 380 or w > umax + 3:
            continue
        z = torch.empty_like(v)
        try:
            hp = (nc, w, LINKS) if LINKS else (nc, w)
            t = timed(lambda: D.ilu0_apply(f, split, v, nx, ny, nz, S, z=z, skew=skew, work=work, hp=hp))
        except Exception as exc:  # noqa: BLE001
            print(f"  hp {hp} upw {upw}: FAILED {exc}", flush=True)
            continue
        print(f"  hp {hp} upw {upw}: {t:.3f} ms  bitwise={torch.equal(z, z_ref)}", flush=True)
