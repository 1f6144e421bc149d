"""NTD apply sweep time vs CTAs per system (1: both level-3 halves on one SM,
2: a cluster of two SMs), config-4 systems.  python tools/ntd_ctas_scan.py [B1,...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09771_b200 import _lib, problems  # noqa: E402
from paper_1909_09771_b200.batch import BatchSolver  # noqa: E402

sizes = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,8").split(",")]
ins = [problems.baseline_config(4, s % 8) for s in range(min(8, max(sizes)))]
nx, ny, nz = ins[0][2]
for B in sizes:
    a = torch.from_numpy(np.stack([ins[s % len(ins)][0] for s in range(B)])).cuda()
    s = BatchSolver(a, nx, ny, nz, groups=1).setup()
    P = s.precond
    row = []
    for c in (1, 2, "2-nosmb"):
        _lib.load().ntd_set_smb(0 if c == "2-nosmb" else 1)
        c_ = 2 if c == "2-nosmb" else c
        def run():
            _lib.call("ntd_apply_slot_ex", _lib.ptr(P.solve), _lib.ptr(P.work), nx, ny, nz, B, None, c_,
                      _lib.stream())
        run()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(3):
            run()
        e[1].record()
        torch.cuda.synchronize()
        row.append(f"{c}:{e[0].elapsed_time(e[1]) / 3:.3f}")
    _lib.load().ntd_set_smb(1)
    print(f"B={B} ntd apply ms by ctas/system:", " ".join(row), flush=True)
    del s, P, a
    torch.cuda.empty_cache()
