"""Remaining properties of the reference suite on the GPU
path: preconditioner ordering on the reference's 50^3 problems
(tests/test_precond_pcg.py:169-180), manufactured solution
(test_precond_pcg.py:121-128), combined-preconditioner symmetry
(test_precond_pcg.py:160-166), the beta identity (test_acceptance.py:113-123),
ILU0 half independence (test_ilu0.py:82-102) and worker invariance (bitwise,
test_acceptance.py:152-165)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ntd():
    import paper_1909_09771_b200 as m
    return m


@pytest.fixture(scope="module")
def ring50(ntd):
    from paper_1909_09771_b200.problem_gen import CoefficientField, GridSpec, assemble
    return assemble(GridSpec(50, 50, 50), CoefficientField.RING)


def test_ordering_combined_ilu0_none(ntd):
    """combined < ILU0 < none in iterations on the skyscraper field, 50^3,
    max 1000 iterations (test_precond_pcg.py:169-180)."""
    from paper_1909_09771_b200.batch import build_precond
    from paper_1909_09771_b200.problem_gen import CoefficientField, GridSpec, assemble
    a = assemble(GridSpec(50, 50, 50), CoefficientField.SKYSCRAPER)
    b = ntd.make_rhs(a, "ones")
    res = {kind: ntd.pcg(a, b, build_precond(a, kind), tol=1e-7, max_iters=1000)[1]
           for kind in ("ntd+ilu0", "ilu0", "none")}
    assert res["ntd+ilu0"].converged
    its = {k: v.iterations for k, v in res.items()}
    assert its["ntd+ilu0"] < its["ilu0"] < its["none"], its


def test_manufactured_solution(ntd, ring50):
    """b = A 1 gives x = 1 to within 100 tol (test_precond_pcg.py:121-128)."""
    a = ring50
    b = ntd.make_rhs(a, "manufactured")
    x, st = ntd.pcg(a, b, ntd.CombinedPrecond(a), tol=1e-8)
    assert st.converged
    assert np.abs(x - 1.0).max() <= 100 * 1e-8


def test_combined_preconditioner_symmetric(ntd):
    """<u, M^-1 v> = <M^-1 u, v> (test_precond_pcg.py:160-166)."""
    from paper_1909_09771_b200.problem_gen import CoefficientField, GridSpec, assemble
    a = assemble(GridSpec(11, 9, 8), CoefficientField.SKYSCRAPER)
    cp = ntd.CombinedPrecond(a)
    rng = np.random.default_rng(4)
    u, v = rng.standard_normal(a.n_rows), rng.standard_normal(a.n_rows)
    lhs, rhs = u @ ntd.combined_apply(cp, v), ntd.combined_apply(cp, u) @ v
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), 1.0)


def test_beta_identity(ntd):
    """compute_beta(apply_inv, u) = w / u with w = apply_inv(u), 0 where u = 0
    (test_acceptance.py:113-123)."""
    from paper_1909_09771_b200.problem_gen import CoefficientField, GridSpec, assemble
    a = assemble(GridSpec(6, 5, 4), CoefficientField.RING)
    pre = ntd.factor_level3(a)
    rng = np.random.default_rng(6)
    u = rng.uniform(0.5, 1.5, a.n_rows)
    u[::7] = 0.0

    def apply_inv(vec):
        return ntd.ntd_apply(pre, vec)

    beta = ntd.compute_beta(apply_inv, u)
    w = apply_inv(u)
    want = np.where(u != 0.0, w / np.where(u != 0.0, u, 1.0), 0.0)
    assert np.abs(beta - want).max() <= 1e-12 * np.abs(want).max()


def test_ilu0_halves_independent(ntd):
    """Changing the rhs of one half leaves the other half's result bitwise
    unchanged (block-diagonal ILU0, test_ilu0.py:82-102)."""
    from paper_1909_09771_b200.problem_gen import CoefficientField, GridSpec, assemble
    a = assemble(GridSpec(12, 10, 8), CoefficientField.SKYSCRAPER)
    f = ntd.build_block_ilu0(a)
    rng = np.random.default_rng(8)
    r = rng.standard_normal(a.n_rows)
    z0 = ntd.ilu0_apply(f, r)
    r2 = r.copy()
    r2[f.split:] = rng.standard_normal(a.n_rows - f.split)
    z1 = ntd.ilu0_apply(f, r2)
    assert np.array_equal(z0[:f.split], z1[:f.split])
    r3 = r.copy()
    r3[:f.split] = rng.standard_normal(f.split)
    z2 = ntd.ilu0_apply(f, r3)
    assert np.array_equal(z0[f.split:], z2[f.split:])


def test_worker_invariance_bitwise(ntd, ring50):
    """Results do not depend on `workers` / `lanes` (the reference's
    worker-invariance tests, test_acceptance.py:152-165): bitwise equal."""
    a = ring50
    b = ntd.make_rhs(a, "ones")
    runs = []
    for workers in (1, 2, 4):
        cp = ntd.CombinedPrecond(a, workers=workers)
        runs.append(ntd.pcg(a, b, cp, tol=1e-7, workers=workers))
    x0, s0 = runs[0]
    for x, st in runs[1:]:
        assert st.iterations == s0.iterations and np.array_equal(x, x0)
        assert st.relres_history == s0.relres_history
