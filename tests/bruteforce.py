"""Brute-force enumeration helpers for the pins (independent of oracle/ and the product).

Everything here is a direct definition: X_j by enumeration of {0,1}^{I_j}
(Def. "Constraint Set Correspondence" P:259-270), Eq. (MM) P:611 by
minimisation over X_j, E^j P:591, (BP) P:561 by enumeration of {0,1}^n.
"""
import itertools

import numpy as np


def all_bits(k):
    return ((np.arange(2 ** k)[:, None] >> np.arange(k)[None, :]) & 1).astype(np.int64)


def row_sat(s, rel, rhs):
    return (s <= rhs) if rel < 0 else (s >= rhs) if rel > 0 else (s == rhs)


def feasible_set(coef, rel, rhs):
    """X_j as an array [|X_j|, k] of 0/1 assignments (bit h = variable h of I_j)."""
    xs = all_bits(len(coef))
    return xs[row_sat(xs @ np.asarray(coef, dtype=np.int64), rel, rhs)]


def energy(X, lam):
    """E^j(lambda) = min_{x in X_j} x^T lambda."""
    return float(np.min(X @ np.asarray(lam, dtype=np.float64)))


def min_marginal(X, lam, h):
    """(m^0, m^1) of Eq. (MM) P:611 for position h; +inf if no x with x_h = beta."""
    v = X @ np.asarray(lam, dtype=np.float64)
    out = []
    for beta in (0, 1):
        sel = X[:, h] == beta
        out.append(float(v[sel].min()) if sel.any() else float("inf"))
    return tuple(out)


def solve_exhaustive(problem):
    """min <c,x> over x in {0,1}^n with all rows satisfied (Eq. BP); n <= 22."""
    n = problem.n_vars
    assert n <= 22
    xs = all_bits(n)
    ok = np.ones(xs.shape[0], dtype=bool)
    for j in range(problem.n_cons):
        v, c, rel, rhs = problem.row(j)
        ok &= row_sat(xs[:, v] @ c.astype(np.int64), rel, rhs)
    if not ok.any():
        return None
    vals = xs[ok] @ problem.cost
    return float(vals.min())


def assignment_opt(cmat):
    """Linear assignment optimum by enumerating permutations."""
    n = cmat.shape[0]
    return min(sum(cmat[a, p[a]] for a in range(n)) for p in itertools.permutations(range(n)))
