"""Golden fixtures for the reference's public single-line / single-plane
factorisations and BLAS-1 helpers (run here only; the GPU box reads the
committed npz).

    python tests/golden/gen_golden_levels.py

Imports ``ntdprecon`` from /root/reference/pkg/src (copied to /tmp: the tree
is read-only and numba caches need a writable dir) and writes
tests/golden/levels_cases.npz:

  level2/<name>/{in,out}  -- factor_level2(PlaneBands, GridSpec(nx, ny, 1))
      (ntd_factor.py:303-333) on planes of the reference's three fields, a
      Neumann checkerboard and random diagonally dominant planes; in = the
      five plane bands (diag, lower1, upper1, lower2, upper2), out = (l1, u1,
      m_recip), at the reference default lanes = 4;
  level1/<name>/{in,out}  -- factor_level1(LineBands) (ntd_factor.py:277-300);
  blas/<n>/{x,y,alpha,axpy,dot,norm2} -- axpy / dot / norm2
      (banded_core.py:133-147) on seeded vectors.
"""

import os
import shutil
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

HERE = os.path.dirname(os.path.abspath(__file__))

_SRC = "/root/reference/pkg/src/ntdprecon"
_DST = "/tmp/golden_ref/ntdprecon"
if not os.path.isdir(_DST):
    shutil.copytree(_SRC, _DST)
sys.path.insert(0, "/tmp/golden_ref")

import numpy as np  # noqa: E402
import ntdprecon as ref  # noqa: E402
from ntdprecon.ntd_factor import LineBands, PlaneBands, factor_level1, factor_level2  # noqa: E402

PLANES = [(1, 2), (2, 2), (5, 4), (9, 7), (13, 11), (16, 16), (33, 20), (40, 3)]


def plane_of(a, k=0):
    nxy = a.nx * a.ny
    sl = slice(k * nxy, (k + 1) * nxy)
    d = a.data
    return np.stack([d[3, sl], d[2, sl], d[4, sl], d[1, sl], d[5, sl]])


def main():
    out = {}
    names = []
    rng = np.random.default_rng(31)
    for nx, ny in PLANES:
        for field in (1, 2, 3):
            a = ref.assemble(ref.GridSpec(nx, ny, 3), field)
            names.append((f"f{field}_{nx}x{ny}", nx, ny, plane_of(a, 1)))
        # random diagonally dominant plane with the grid's zero pattern
        nxy = nx * ny
        bands = np.zeros((5, nxy))
        i = np.arange(nxy) % nx
        j = np.arange(nxy) // nx
        bands[1] = np.where(i > 0, -rng.uniform(0.1, 1.0, nxy), 0.0)
        bands[2] = np.where(i < nx - 1, -rng.uniform(0.1, 1.0, nxy), 0.0)
        bands[3] = np.where(j > 0, -rng.uniform(0.1, 1.0, nxy), 0.0)
        bands[4] = np.where(j < ny - 1, -rng.uniform(0.1, 1.0, nxy), 0.0)
        bands[0] = 4.5 + rng.uniform(0.0, 1.0, nxy)
        names.append((f"rand_{nx}x{ny}", nx, ny, bands))
    keys = []
    for name, nx, ny, b in names:
        l1, u1, mr = factor_level2(PlaneBands(*[np.ascontiguousarray(v) for v in b]), ref.GridSpec(nx, ny, 1))
        out[f"level2/{name}/in"] = b
        out[f"level2/{name}/grid"] = np.array([nx, ny])
        out[f"level2/{name}/out"] = np.stack([l1, u1, mr])
        keys.append(name)
    out["level2_names"] = np.array(keys)
    lkeys = []
    for n in (1, 2, 3, 7, 32, 33, 96, 97):
        d = 2.2 + rng.uniform(0, 1, n)
        lo = -rng.uniform(0.1, 1.0, n)
        up = -rng.uniform(0.1, 1.0, n)
        lo[0] = 0.0
        up[-1] = 0.0
        mr = factor_level1(LineBands(d, lo, up))
        out[f"level1/{n}/in"] = np.stack([d, lo, up])
        out[f"level1/{n}/out"] = mr
        lkeys.append(n)
    out["level1_sizes"] = np.array(lkeys)
    for n in (1, 2, 17, 1000, 20011):
        x = rng.standard_normal(n)
        y = rng.standard_normal(n)
        alpha = float(rng.standard_normal())
        out[f"blas/{n}/x"] = x
        out[f"blas/{n}/y"] = y
        out[f"blas/{n}/alpha"] = np.array([alpha])
        out[f"blas/{n}/axpy"] = ref.axpy(alpha, x, y)
        out[f"blas/{n}/dot"] = np.array([ref.dot(x, y)])
        out[f"blas/{n}/norm2"] = np.array([ref.norm2(x)])
    out["blas_sizes"] = np.array([1, 2, 17, 1000, 20011])
    np.savez_compressed(os.path.join(HERE, "levels_cases.npz"), **out)
    print(len(keys), "planes,", len(lkeys), "lines")


if __name__ == "__main__":
    main()
