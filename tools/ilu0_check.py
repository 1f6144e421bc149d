"""Skew ILU0 apply vs the C oracle on small random grids (debug aid; run
under compute-sanitizer to catch out-of-bounds accesses)."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402
import paper_1909_09771_b200 as ntd  # noqa: E402
from paper_1909_09771_b200 import problems  # noqa: E402

for (nx, ny, nz) in [(5, 4, 6), (12, 12, 12), (40, 35, 8), (33, 70, 4)]:
    rng = np.random.default_rng(1)
    kap = np.exp(rng.normal(0, 1, (nz, ny, nx)))
    data = problems.assemble_kappa(kap, nx, ny, nz)
    a = ntd.BandedMatrix(nx, ny, nz, data)
    g = ntd.build_block_ilu0(a)
    f, split = oracle.build_block_ilu0(data, nx, ny, nz)
    r = rng.uniform(-1, 1, nx * ny * nz)
    ok = np.array_equal(ntd.ilu0_apply(g, r), oracle.ilu0_apply(f, split, r, nx, ny, nz))
    print((nx, ny, nz), "skew" if g.skew() is not None else "ref-layout", "bitwise" if ok else "MISMATCH")

if os.environ.get("NTD_LIB_OVERRIDE", "").endswith("_chk.so"):
    import ctypes
    from paper_1909_09771_b200 import _lib
    buf = (ctypes.c_longlong * 6)()
    _lib.load().ntd_skew_check(buf)
    print("first out-of-bounds access (what, block, warp, lane, offset, count):", list(buf))
