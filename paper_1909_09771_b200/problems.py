"""Problem inputs: the reference's coefficient fields and the BASELINE configs.

Setup-time input generation only (not on the solve path).  ``assemble_kappa``
restates the reference finite-volume assembly ``_assemble_kernel``
(/root/reference/pkg/src/ntdprecon/problem_gen.py:87-133) with the same
operation order -- harmonic face mean ``2*kc*kn/(kc+kn)``, diagonal summed
x-,x+,y-,y+,z-,z+ -- generalised to per-face Dirichlet/Neumann flags (a
Neumann face adds nothing, a Dirichlet face adds the cell's kappa to the
diagonal).  ``reference_kappa`` restates ``_kappa_scalar``/``_kappa_grid``
(problem_gen.py:42-84).  ``baseline_config`` builds the five BASELINE.json
configs from the seeded recipe of SURVEY.md section 8(d) (synthetic inputs:
the reference publishes no dataset).
"""

import numpy as np

ALL_DIRICHLET = (True, True, True, True, True, True)


def assemble_kappa(kappa, nx, ny, nz, dirichlet=ALL_DIRICHLET):
    """7-band matrix (7, N) for a cellwise kappa array indexed [k][j][i]."""
    kap = np.ascontiguousarray(kappa, dtype=np.float64).reshape(nz, ny, nx)
    n = nx * ny * nz
    data = np.zeros((7, nz, ny, nx))
    diag = np.zeros((nz, ny, nx))
    xm, xp, ym, yp, zm, zp = (bool(f) for f in dirichlet)

    def face(kc, kn):
        return 2.0 * kc * kn / (kc + kn)

    # order matters for bitwise parity: x-, x+, y-, y+, z-, z+ (problem_gen.py:98-122)
    if nx > 1:
        c = face(kap[:, :, 1:], kap[:, :, :-1])
        data[2, :, :, 1:] = -c
        diag[:, :, 1:] += c
    if xm:
        diag[:, :, 0] += kap[:, :, 0]
    if nx > 1:
        c = face(kap[:, :, :-1], kap[:, :, 1:])
        data[4, :, :, :-1] = -c
        diag[:, :, :-1] += c
    if xp:
        diag[:, :, -1] += kap[:, :, -1]
    if ny > 1:
        c = face(kap[:, 1:, :], kap[:, :-1, :])
        data[1, :, 1:, :] = -c
        diag[:, 1:, :] += c
    if ym:
        diag[:, 0, :] += kap[:, 0, :]
    if ny > 1:
        c = face(kap[:, :-1, :], kap[:, 1:, :])
        data[5, :, :-1, :] = -c
        diag[:, :-1, :] += c
    if yp:
        diag[:, -1, :] += kap[:, -1, :]
    if nz > 1:
        c = face(kap[1:], kap[:-1])
        data[0, 1:] = -c
        diag[1:] += c
    if zm:
        diag[0] += kap[0]
    if nz > 1:
        c = face(kap[:-1], kap[1:])
        data[6, :-1] = -c
        diag[:-1] += c
    if zp:
        diag[-1] += kap[-1]
    data[3] = diag
    return data.reshape(7, n)


def reference_kappa(field, nx, ny, nz):
    """problem_gen.py:42-84: Types 1 (skyscraper), 2 (ring), 3 (Poisson)."""
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    x = (i + 0.5) / nx
    y = (j + 0.5) / ny
    z = (k + 0.5) / nz
    kap = np.ones((nz, ny, nx))
    if int(field) == 1:
        ix = np.floor(10.0 * x).astype(np.int64)
        iy = np.floor(10.0 * y).astype(np.int64)
        iz = np.floor(10.0 * z).astype(np.int64)
        hi = (ix % 2 == 0) & (iy % 2 == 0) & (iz % 2 == 0)
        kap[hi] = 1.0e3 * (iy[hi] + 1.0)
    elif int(field) == 2:
        dx, dy, dz = x - 0.5, y - 0.5, z - 0.5
        r = np.sqrt(dx * dx + dy * dy + dz * dz)
        ring = (1.0 / (2.0 * np.sqrt(2.0)) <= r) & (r <= 0.5)
        kap[ring] = 1.0e3
    elif int(field) != 3:
        raise ValueError(f"unknown coefficient field {field!r}")
    return kap


CONFIGS = {
    1: dict(name="cfg1-poisson-32", grid=(32, 32, 32), batch=1),
    2: dict(name="cfg2-checker-64-neumann", grid=(64, 64, 64), batch=1),
    3: dict(name="cfg3-layered-128", grid=(128, 128, 128), batch=1),
    4: dict(name="cfg4-batch64-lognormal-96", grid=(96, 96, 96), batch=64),
    5: dict(name="cfg5-randcubes-350", grid=(350, 350, 350), batch=1),
}


def baseline_kappa(cfg, system=0):
    """Seeded kappa field [k][j][i], Dirichlet flags and the rng positioned for
    x_true (default_rng(1000*cfg + s), kappa draws first)."""
    nx, ny, nz = CONFIGS[cfg]["grid"]
    rng = np.random.default_rng(1000 * cfg + system)
    bc = ALL_DIRICHLET
    if cfg == 1:
        kap = np.ones((nz, ny, nx))
    elif cfg == 2:
        k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        odd = ((i // 8) + (j // 8) + (k // 8)) % 2 == 1
        kap = np.where(odd, 1.0e3, 1.0)
        bc = (False, False, False, False, True, False)
    elif cfg == 3:
        u = rng.uniform(-4.0, 4.0, 8)
        kap = np.repeat(10.0 ** u, 16)[:, None, None] * np.ones((1, ny, nx))
    elif cfg == 4:
        g = rng.normal(0.0, 2.0, (24, 24, 24))
        kap = np.exp(g).repeat(4, 0).repeat(4, 1).repeat(4, 2)
    elif cfg == 5:
        c = rng.integers(0, 3, (10, 10, 10))
        vals = np.array([1.0e-3, 1.0, 1.0e3])[c]
        kap = vals.repeat(35, 0).repeat(35, 1).repeat(35, 2)
    else:
        raise ValueError(f"unknown config {cfg}")
    return np.ascontiguousarray(kap), bc, rng


def baseline_config(cfg, system=0):
    """Returns (data (7,N), x_true (N,), (nx,ny,nz)); b = A x_true is formed by
    the caller with the product spmv (bitwise equal to the reference's)."""
    nx, ny, nz = CONFIGS[cfg]["grid"]
    kap, bc, rng = baseline_kappa(cfg, system)
    data = assemble_kappa(kap, nx, ny, nz, bc)
    x_true = rng.uniform(-1.0, 1.0, nx * ny * nz)
    return data, x_true, (nx, ny, nz)
