"""The two-sided line solve of the GPU apply (csrc/ntd_line_ts.cuh,
ts::k_solve_ts in csrc/ntd_apply_ts.cuh), restated in numpy and checked on the
CPU against the oracle's twisted line solve (the reference's _line_solve,
ntd_solve.py:107-137): same operator, rounding-level difference only.

  T of a factored line: sub-diagonal l1, super-diagonal u1, twisted pivots
  1 / m_recip with the twist at t = (n - 1) // 2 (ntd_factor.py:86-110).
  delta / gamma: pivots of the elimination carried from the first / last cell
  across the whole line; 1 / mu_j = delta_j + gamma_j - d_j is the twisted
  pivot at cell j; x_j = mu_j (f_j + g_j - r_j) with f / g the rhs eliminated
  from the first / last cell.  The kernel works on the scaled quantities
  rho = mu r, f' = mu f, g' = mu g with multipliers eF, eB.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import oracle  # noqa: E402


def solve_records(l1, u1, mr):
    """eF, eB, mu of one line from its factor (what ts::k_solve_ts stores)."""
    n = len(mr)
    t = (n - 1) // 2
    d = 1.0 / mr
    for c in range(n):
        if 0 < c <= t:
            d[c] += (l1[c] * u1[c - 1]) * mr[c - 1]
        if t <= c < n - 1:
            d[c] += (u1[c] * l1[c + 1]) * mr[c + 1]
    de = 1.0 / mr
    for c in range(t, n):
        de[c] = d[c] - (l1[c] * u1[c - 1]) / de[c - 1] if c > 0 else d[c]
    ga = 1.0 / mr
    for c in range(t, -1, -1):
        ga[c] = d[c] - (u1[c] * l1[c + 1]) / ga[c + 1] if c < n - 1 else d[c]
    nu = de + ga - d
    nu[t] = 1.0 / mr[t]
    mu = 1.0 / nu
    mu[t] = mr[t]
    eF = np.zeros(n)
    eB = np.zeros(n)
    eF[1:] = -(l1[1:] * nu[:-1]) / (de[:-1] * nu[1:])
    eB[:-1] = -(u1[:-1] * nu[1:]) / (ga[1:] * nu[:-1])
    return eF, eB, mu


def two_sided(eF, eB, mu, r):
    rho = mu * r
    f = np.empty_like(rho)
    g = np.empty_like(rho)
    acc = 0.0
    for j in range(len(rho)):
        acc = rho[j] + eF[j] * acc
        f[j] = acc
    acc = 0.0
    for j in range(len(rho) - 1, -1, -1):
        acc = rho[j] + eB[j] * acc
        g[j] = acc
    return f + g - rho


def line_operator(n, rng, jump):
    """A one-line BandedMatrix (7, n): diffusion with coefficient jumps and a positive shift."""
    k = 10.0 ** rng.uniform(-jump, jump, n + 1)
    data = np.zeros((7, n))
    data[2, 1:] = -k[1:n]
    data[4, :-1] = -k[1:n]
    data[3] = k[:-1] + k[1:] + 10.0 ** rng.uniform(-3, 0, n)
    return data


@pytest.mark.parametrize("n", [1, 2, 3, 4, 17, 32, 33, 96, 350])
@pytest.mark.parametrize("jump", [0.0, 3.0])
def test_two_sided_equals_twisted_line_solve(n, jump):
    rng = np.random.default_rng(100 * n + int(jump))
    data = line_operator(n, rng, jump)
    pre = oracle.factor_level3(data, n, 1, 1)
    eF, eB, mu = solve_records(pre[0].copy(), pre[1].copy(), pre[6].copy())
    assert eF[0] == 0.0 and eB[-1] == 0.0  # the kernel's edge lanes rely on these exact zeros
    for _ in range(3):
        r = rng.uniform(-1, 1, n)
        x_ref = oracle.ntd_apply(pre, r, n, 1, 1)
        x = two_sided(eF, eB, mu, r)
        # (with jumps of 10^6 between cells the line's condition number reaches 3e5: both solves are then
        # 2-3e-12 from the exact solution, and from each other; the bar of the apply is 1e-10)
        tol = 1e-13 if jump == 0.0 else 2e-11
        assert np.abs(x - x_ref).max() <= tol * np.abs(x_ref).max(), (n, jump)


def test_twist_pivot_is_the_references():
    """At the twist cell mu is the stored m_recip itself, and left / right of it the
    forward / backward pivots are the stored ones (1 / m_recip)."""
    rng = np.random.default_rng(7)
    n = 41
    pre = oracle.factor_level3(line_operator(n, rng, 2.0), n, 1, 1)
    _, _, mu = solve_records(pre[0].copy(), pre[1].copy(), pre[6].copy())
    assert mu[(n - 1) // 2] == pre[6][(n - 1) // 2]
    assert np.all(mu > 0)
