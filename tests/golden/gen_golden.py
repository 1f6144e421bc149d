"""Generate golden fixtures from the REAL reference package (run here only).

    python tests/golden/gen_golden.py

Imports ``ntdprecon`` from /root/reference/pkg/src (copied to /tmp because the
tree is read-only and numba caches need a writable dir), runs its public API on
seeded inputs and writes:

  tests/golden/small_cases.npz  -- full arrays for small grids (A, factored
      bands, ntd_apply, ILU0 factors/apply, combined apply, PCG iterations and
      relres history) for the reference's three fields and the BASELINE-style
      fields (Neumann checkerboard, layered, log-normal, random cubes);
  tests/golden/configs.json     -- BASELINE config 1/2 fingerprints (fsum of
      bands and of an apply, sampled entries) and the reference's PCG
      iteration counts / relres histories at tol 1e-8.

The GPU box has no /root/reference; tests read only these committed files.
"""

import json
import zlib
import math
import os
import shutil
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

_SRC = "/root/reference/pkg/src/ntdprecon"
_DST = "/tmp/golden_ref/ntdprecon"
if not os.path.isdir(_DST):
    shutil.copytree(_SRC, _DST)
sys.path.insert(0, "/tmp/golden_ref")

import numpy as np  # noqa: E402
import ntdprecon as ref  # noqa: E402

from paper_1909_09771_b200 import problems  # noqa: E402

SMALL_GRIDS = [(1, 1, 1), (1, 1, 5), (4, 1, 1), (1, 3, 1), (2, 2, 2), (3, 4, 5),
               (5, 3, 4), (2, 7, 3), (6, 6, 6), (7, 5, 9), (10, 9, 8), (13, 11, 12)]


def small_systems():
    for g in SMALL_GRIDS:
        for field in (1, 2, 3):
            a = ref.assemble(ref.GridSpec(*g), field)
            yield f"g{g[0]}x{g[1]}x{g[2]}_f{field}", g, a.data
    rng = np.random.default_rng(777)
    for g in [(8, 8, 8), (12, 10, 9), (16, 16, 16)]:
        nx, ny, nz = g
        k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        cheq = np.where(((i // 4) + (j // 4) + (k // 4)) % 2 == 1, 1.0e3, 1.0)
        yield (f"g{nx}x{ny}x{nz}_checker_neumann", g,
               problems.assemble_kappa(cheq, nx, ny, nz, (False,) * 4 + (True, False)))
        lay = np.repeat(10.0 ** rng.uniform(-4, 4, nz), ny * nx).reshape(nz, ny, nx)
        yield f"g{nx}x{ny}x{nz}_layered", g, problems.assemble_kappa(lay, nx, ny, nz)
        logn = np.exp(rng.normal(0.0, 2.0, (nz, ny, nx)))
        yield f"g{nx}x{ny}x{nz}_lognormal", g, problems.assemble_kappa(logn, nx, ny, nz)
        cub = np.array([1e-3, 1.0, 1e3])[rng.integers(0, 3, (nz, ny, nx))]
        yield f"g{nx}x{ny}x{nz}_cubes", g, problems.assemble_kappa(cub, nx, ny, nz)


def run_case(name, g, data, out):
    nx, ny, nz = g
    n = nx * ny * nz
    a = ref.BandedMatrix(nx, ny, nz, data)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    v = rng.uniform(-1.0, 1.0, n)
    out[name + "/A"] = a.data
    out[name + "/v"] = v
    out[name + "/spmv"] = ref.spmv(a, v)
    pre = ref.factor_level3(a)
    out[name + "/pre"] = np.stack([pre.l1, pre.u1, pre.l2, pre.u2, pre.l3,
                                   pre.u3, pre.m_recip])
    out[name + "/ntd"] = ref.ntd_apply(pre, v)
    out[name + "/ntd_lanes1"] = ref.ntd_apply(pre, v, lanes=1)
    if n >= 2:
        ilu = ref.build_block_ilu0(a)
        out[name + "/ilu"] = ilu.data
        out[name + "/ilu_split"] = np.array([ilu.split])
        out[name + "/ilu_apply"] = ref.ilu0_apply(ilu, v)
        cp = ref.CombinedPrecond(a)
        out[name + "/combined"] = ref.combined_apply(cp, v)
        b = ref.spmv(a, v)
        x, st = ref.pcg(a, b, cp, tol=1e-8, max_iters=100)
        out[name + "/pcg_x"] = x
        out[name + "/pcg_hist"] = np.array(st.relres_history)
        out[name + "/pcg_iters"] = np.array([st.iterations, int(st.converged)])
        x0, st0 = ref.pcg(a, b, None, tol=1e-8, max_iters=400)
        out[name + "/cg_iters"] = np.array([st0.iterations, int(st0.converged)])


def fingerprint(arr, idx):
    return {"fsum": math.fsum(np.asarray(arr).ravel().tolist()),
            "sample": [float(arr[i]) for i in idx]}


def config_case(cfg):
    data, x_true, (nx, ny, nz) = problems.baseline_config(cfg)
    a = ref.BandedMatrix(nx, ny, nz, data)
    n = a.n_rows
    b = ref.spmv(a, x_true)
    idx = np.random.default_rng(cfg).integers(0, n, 64).tolist()
    pre = ref.factor_level3(a)
    rec = {"grid": [nx, ny, nz], "sample_idx": idx,
           "b": fingerprint(b, idx)}
    for name in ("l1", "u1", "l2", "u2", "m_recip"):
        rec["pre_" + name] = fingerprint(getattr(pre, name), idx)
    v = np.random.default_rng(100 + cfg).uniform(-1.0, 1.0, n)
    rec["apply_v_seed"] = 100 + cfg
    rec["ntd_apply"] = fingerprint(ref.ntd_apply(pre, v), idx)
    ilu = ref.build_block_ilu0(a)
    rec["ilu_apply"] = fingerprint(ref.ilu0_apply(ilu, v), idx)
    cp = ref.CombinedPrecond(a)
    rec["combined"] = fingerprint(ref.combined_apply(cp, v), idx)
    x, st = ref.pcg(a, b, cp, tol=1e-8, max_iters=200)
    rec["pcg_iters"] = st.iterations
    rec["pcg_converged"] = bool(st.converged)
    rec["pcg_hist"] = st.relres_history
    rec["pcg_err_vs_xtrue"] = float(np.linalg.norm(x - x_true) / np.linalg.norm(x_true))
    return rec


def main():
    out = {}
    names = []
    for name, g, data in small_systems():
        run_case(name, g, data, out)
        names.append(name)
        print("case", name, flush=True)
    out["names"] = np.array(names)
    # chain / twist / level-1/2 known answers
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 8, 9, 33):
        dr = rng.uniform(0.5, 1.5, n)
        off = rng.uniform(-0.4, 0.4, n)
        bb = rng.uniform(-1, 1, n)
        for direction in ("forward", "backward"):
            for lanes in (1, 4):
                key = f"chain/{n}/{direction}/{lanes}"
                out[key] = ref.chain_bidiagonal_solve(dr, off, bb, direction, lanes)
        out[f"chain/{n}/in"] = np.stack([dr, off, bb])
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **out)
    cfgs = {str(c): config_case(c) for c in (1, 2)}
    with open(os.path.join(HERE, "configs.json"), "w") as fh:
        json.dump(cfgs, fh, indent=1)
    print({c: (v["pcg_iters"], v["pcg_hist"][-1]) for c, v in cfgs.items()})


if __name__ == "__main__":
    main()
