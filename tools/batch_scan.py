"""Per-kernel device time vs batch size on config-4 systems (profiling aid).

    python tools/batch_scan.py [B1,B2,...]

For each batch size: NTD apply, ILU0 apply (skew + conversions), residual
(t = r - A w), and the PCG iteration kernels, CUDA-event timed on the current
stream, median of 5.  Shows which kernels are latency-bound (flat in B) and
which are bandwidth-bound (linear in B).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402
from paper_1909_09771_b200.batch import BatchSolver  # noqa: E402


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        fn()
        e[1].record()
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    return float(np.median(ts))


sizes = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16,32,64").split(",")]
cfg = int(os.environ.get("SCAN_CFG", "4"))
Bmax = max(sizes)
ins = [problems.baseline_config(cfg, s) for s in range(Bmax if cfg == 4 else 1)]
nx, ny, nz = ins[0][2]
n = nx * ny * nz
out = []
for B in sizes:
    a = torch.from_numpy(np.stack([ins[s % len(ins)][0] for s in range(B)])).cuda()
    xt = torch.from_numpy(np.stack([ins[s % len(ins)][1] for s in range(B)])).cuda()
    b = torch.empty_like(xt)
    _lib.call("ntd_spmv", _lib.ptr(a), _lib.ptr(xt), _lib.ptr(b), nx, ny, nz, B, None, _lib.stream())
    s = BatchSolver(a, nx, ny, nz, groups=1).setup()
    P = s.precond
    v = torch.rand_like(b)
    x = torch.empty_like(b)
    z = torch.empty_like(b)
    P.apply(v, z)  # allocates scratch
    row = {"B": B}
    row["ntd_apply"] = timed(lambda: D.ntd_apply(P.pre, v, nx, ny, nz, B, x=x, work=P.work, solve=P.solve))
    row["ilu0_apply"] = timed(lambda: D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, B, z=x, skew=P.skew,
                                                   work=P.skew_work, ctas=P.ilu_ctas))
    row["residual"] = timed(lambda: D.residual(a, v, x, nx, ny, nz, B, t=z))
    row["combined"] = timed(lambda: P.apply(v, z))
    res = s.solve(b)
    it = max(res.iterations)
    row["solve_ms"] = timed(lambda: s.solve(b), reps=3)
    row["iters_max"] = it
    row["ms_per_iter"] = row["solve_ms"] / it
    row["munk_iter_s"] = n * sum(res.iterations) / (row["solve_ms"] / 1e3) / 1e6
    print(json.dumps(row), flush=True)
    out.append(row)
    del s, P, a, xt, b, v, x, z
    torch.cuda.empty_cache()
