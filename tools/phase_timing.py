"""Where a stream group's PCG iteration spends its time inside the batched
config-4 solve: an event is recorded on the group's stream after every
native call, so each interval is (queueing for SMs + run time) of that call.
python tools/phase_timing.py [systems] [groups]"""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200 import device as D  # noqa: E402
from paper_1909_09771_b200.batch import BatchSolver  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
G = int(sys.argv[2]) if len(sys.argv) > 2 else None
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
solver = BatchSolver(a, nx, ny, nz, max_iters=200, groups=G).setup()
for _ in range(2):
    solver.solve(b)
torch.cuda.synchronize()

marks = []  # (stream id, name, event)
orig = _lib.call


def traced(name, *args):
    rc = orig(name, *args)
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    marks.append((torch.cuda.current_stream().cuda_stream, name, ev))
    return rc


_lib.call = traced
import paper_1909_09771_b200.device as Dm  # noqa: E402
Dm._lib.call = traced
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = solver.solve(b)
e1.record()
torch.cuda.synchronize()
total = e0.elapsed_time(e1)
per_stream = collections.defaultdict(list)
for sid, name, ev in marks:
    per_stream[sid].append((name, ev))
acc = collections.defaultdict(float)
cnt = collections.Counter()
span = []
for sid, lst in per_stream.items():
    prev = None
    for name, ev in lst:
        if prev is not None:
            acc[name] += prev.elapsed_time(ev)
            cnt[name] += 1
        prev = ev
    span.append(lst[0][1].elapsed_time(lst[-1][1]))
its = sum(res.iterations)
print(f"systems {S} groups {len(solver.groups)} solve {total:.1f} ms, iterations mean {its / S:.2f} max {max(res.iterations)}")
print(f"group spans ms: min {min(span):.1f} max {max(span):.1f}")
tot = sum(acc.values())
for name in sorted(acc, key=lambda k: -acc[k]):
    print(f"  {name:32s} {acc[name] / cnt[name]:8.3f} ms/call x {cnt[name]:5d}  share {acc[name] / tot:6.1%}")
