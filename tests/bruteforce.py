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


def lifted_passes(problem, directions, omega=0.5, clamp=None):
    """Enumeration implementation of the appendix's lifted representation
    (update P:53-56 read as A8, infinite sides clamped as A5):
    per BDD j two costs per variable, lambda^{j,0} = 0 and lambda^{j,1} =
    c_i/|J_i|; a pass visits the hops in order and, at hop h,
    m^beta = min over x in X_j with x_h = beta of sum_t lambda^{j, x_t}_t
    (at the visit-time costs, A3), d = clamp(m^1 - m^0), then
      lambda^{j,b} += -omega max(d_b, 0) + (omega/|J_i|) sum_k max(dbar_b, 0)
    with d_1 = d, d_0 = -d.  Yields (lambda^0, lambda^1, bound, delta_bar)
    after each pass, slots in canonical order; the bound is the plain sum of
    per-BDD minima plus the free term.  No BDDs, no shortest paths."""
    rows = [problem.row(j) for j in range(problem.n_cons)]
    X = [feasible_set(c, r, b) for (_, c, r, b) in rows]
    deg = np.bincount(problem.col_var, minlength=problem.n_vars)
    if clamp is None:
        clamp = 1e4 * (1.0 + float(np.abs(problem.cost).max()))
    l1 = [problem.cost[v] / deg[v] for (v, _, _, _) in rows]
    l0 = [np.zeros(len(v)) for (v, _, _, _) in rows]
    dbar = [np.zeros(len(v)) for (v, _, _, _) in rows]
    free = sum(min(problem.cost[i], 0.0) for i in range(problem.n_vars) if deg[i] == 0)
    for fwd in directions:
        ap = np.zeros(problem.n_vars)
        an = np.zeros(problem.n_vars)
        for j, (v, _, _, _) in enumerate(rows):  # j ascending (A1)
            for h, i in enumerate(v):
                ap[i] += max(dbar[j][h], 0.0)
                an[i] += max(-dbar[j][h], 0.0)
        ap = np.divide(ap, deg, out=np.zeros_like(ap), where=deg > 0)
        an = np.divide(an, deg, out=np.zeros_like(an), where=deg > 0)
        new = []
        for j, (v, _, _, _) in enumerate(rows):
            k = len(v)
            dl = np.zeros(k)
            for h in (range(k) if fwd else reversed(range(k))):
                vals = X[j] @ l1[j] + (1 - X[j]) @ l0[j]
                m = []
                for beta in (0, 1):
                    sel = vals[X[j][:, h] == beta]
                    m.append(sel.min() if sel.size else np.inf)
                if np.isinf(m[1]):
                    d = clamp
                elif np.isinf(m[0]):
                    d = -clamp
                else:
                    d = m[1] - m[0]
                dl[h] = omega * d
                l1[j][h] = (l1[j][h] - max(dl[h], 0.0)) + ap[v[h]]
                l0[j][h] = (l0[j][h] - max(-dl[h], 0.0)) + an[v[h]]
            new.append(dl)
        dbar = new
        lb = sum(float(np.min(X[j] @ l1[j] + (1 - X[j]) @ l0[j])) for j in range(len(rows))) + free
        yield (np.concatenate(l0) if l0 else np.zeros(0), np.concatenate(l1) if l1 else np.zeros(0), lb,
               np.concatenate(dbar) if dbar else np.zeros(0))
