"""Repeated graphed pcg() solves on one CombinedPrecond: histories, iterations and x must repeat."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_09771_b200 as ntd  # noqa: E402
from paper_1909_09771_b200 import problems  # noqa: E402

data, xt, g = problems.baseline_config(1)
a = ntd.BandedMatrix(*g, data)
b = ntd.spmv(a, xt)
cp = ntd.CombinedPrecond(a)
for k in range(3):
    x, st = ntd.pcg(a, b, cp, tol=1e-8)
    print(k, st.iterations, st.final_relres, st.relres_history[:3], float(np.abs(x - xt).max()))
bd = torch.from_numpy(b).cuda()
for k in range(2):
    x, st = ntd.pcg(a, bd, cp, tol=1e-8)
    print("dev", k, st.iterations, st.final_relres, st.relres_history[:3])
