"""BASELINE config generator (paper_1909_09771_b200/problems.py) against the
reference-run fingerprints of SURVEY.md 8(d) (math.fsum of kappa, x_true, b)
and against the reference assembly on its own fields."""

import math

import numpy as np
import pytest

import oracle
from conftest import grid_of
from paper_1909_09771_b200 import problems

FINGERPRINTS = {  # cfg, system: (sum kappa, sum x_true, sum b, x_true[0], x_true[1])
    (1, 0): (32768.0, -7.6248236803146305, 22.426705795024812, 0.042771475950125426, 0.20768369401265918),
    (2, 0): (131203072.0, -571.3660277988912, 20347.88949814478, 0.15027263771527255, 0.3128492185857741),
    (3, 0): (325658178.2418348, 445.79308278399304, 16853.13433005271, 0.5584083346409148, -0.13241338240039435),
    (4, 0): (6575985.021940704, 72.7935318478414, -2006.9336192187773, 0.7562091185828781, 0.7617643380875208),
    (4, 63): (6290951.540888283, -796.6623764744613, 1668.1373715058744, None, None),
}


@pytest.mark.parametrize("cfg,s", sorted(FINGERPRINTS))
def test_baseline_fingerprints(cfg, s):
    kap, bc, rng = problems.baseline_kappa(cfg, s)
    data, x_true, (nx, ny, nz) = problems.baseline_config(cfg, s)
    b = oracle.spmv(data, x_true, nx, ny, nz)
    fk, fx, fb, x0, x1 = FINGERPRINTS[(cfg, s)]
    assert math.fsum(kap.ravel()) == fk
    assert math.fsum(x_true) == fx
    assert math.fsum(b) == fb
    if x0 is not None:
        assert (x_true[0], x_true[1]) == (x0, x1)


@pytest.mark.slow
def test_config5_fingerprint():
    kap, bc, rng = problems.baseline_kappa(5)
    assert math.fsum(kap.ravel()) == 14549473255.625


def test_reference_fields_assembly_bitwise(golden):
    for name in [str(n) for n in golden["names"]]:
        if not name.endswith(("_f1", "_f2", "_f3")):
            continue
        nx, ny, nz = grid_of(name)
        kap = problems.reference_kappa(int(name[-1]), nx, ny, nz)
        assert np.array_equal(problems.assemble_kappa(kap, nx, ny, nz), golden[name + "/A"]), name


def test_neumann_faces_add_nothing():
    kap = np.full((3, 3, 3), 2.0)
    d_all = problems.assemble_kappa(kap, 3, 3, 3)
    d_neu = problems.assemble_kappa(kap, 3, 3, 3, (False,) * 6)
    # interior cell: identical; corner cell loses 3 Dirichlet contributions
    assert d_all[3, 13] == d_neu[3, 13] == 12.0
    assert d_all[3, 0] - d_neu[3, 0] == 6.0
    # Neumann-everywhere operator annihilates constants
    assert np.allclose(oracle.spmv(d_neu, np.ones(27), 3, 3, 3), 0.0)
