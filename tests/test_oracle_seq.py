"""Pins of the oracle's non-deferred (sequential) min-marginal averaging
(with mbar <- m the update (dual_update) is the one of
[lange2021efficient]), -m "not gpu".

Independent reference: `_seq_pass_enum` below re-implements the pass from
its definition -- variables in ascending (descending) order, every min-marginal
by enumeration of X_j (Eq. (MM) P:611 over Def. P:259-270, tests/bruteforce.py)
at the multipliers current at that moment -- with no BDD and no shortest path.
Also pinned: dual feasibility after every pass (P:10 with mbar = m), a
non-decreasing bound, bound <= brute-force OPT.
"""
import numpy as np
import pytest

import synth
from tests import bruteforce as bf


def _clamp(problem):
    return 1e4 * (1.0 + float(np.max(np.abs(problem.cost))))


def _seq_pass_enum(problem, lam, forward, omega, clamp):
    """One non-deferred pass by enumeration; lam: canonical slot array, updated in place."""
    rows = [problem.row(j) for j in range(problem.n_cons)]
    X = [bf.feasible_set(c, rel, rhs) for (v, c, rel, rhs) in rows]
    base = np.concatenate([[0], np.cumsum([len(r[0]) for r in rows])]).astype(int)
    slots_of = {}
    for j, (v, c, rel, rhs) in enumerate(rows):
        for h, i in enumerate(v):
            slots_of.setdefault(int(i), []).append((j, h))
    order = range(problem.n_vars) if forward else range(problem.n_vars - 1, -1, -1)
    for i in order:
        if i not in slots_of:
            continue
        dl = []
        for (j, h) in slots_of[i]:  # j ascending
            m0, m1 = bf.min_marginal(X[j], lam[base[j]:base[j + 1]], h)
            d = clamp if np.isinf(m1) else (-clamp if np.isinf(m0) else m1 - m0)
            dl.append(omega * d)
        avg = sum(dl) / len(dl)
        for (j, h), d in zip(slots_of[i], dl):
            lam[base[j] + h] = lam[base[j] + h] - d + avg
    return lam


def _raw_bound(problem, lam):
    e = 0.0
    base = 0
    for j in range(problem.n_cons):
        v, c, rel, rhs = problem.row(j)
        e += bf.energy(bf.feasible_set(c, rel, rhs), lam[base:base + len(v)])
        base += len(v)
    deg = np.bincount(problem.col_var, minlength=problem.n_vars)
    return e + float(np.minimum(problem.cost[deg == 0], 0).sum())


def _feasibility(problem, lam):
    s = np.zeros(problem.n_vars)
    np.add.at(s, problem.col_var, lam)
    deg = np.bincount(problem.col_var, minlength=problem.n_vars)
    return float(np.max(np.abs(s - problem.cost)[deg > 0], initial=0.0))


@pytest.mark.parametrize("omega", [0.5, 1.0, 0.3])
def test_seq_pass_matches_enumeration(oracle_mod, omega):
    """Every pass of oracle_pass_seq equals the definition-level enumeration."""
    for seed in range(40):
        p = synth.random_ilp(300 + seed, n=9, m=6, kmax=6, coef=3, forced_ok=seed % 4 == 0)
        o = oracle_mod.Oracle(p)
        lam = o.lam().copy()
        for t in range(4):
            fwd = t % 2 == 0
            o.pass_seq(fwd, omega)
            _seq_pass_enum(p, lam, fwd, omega, _clamp(p))
            assert np.max(np.abs(o.lam() - lam)) <= 1e-9 * (1 + np.abs(lam).max()), (seed, t)


def test_seq_invariants_and_bound(oracle_mod):
    """Feasible after every pass (no deferred term), bound = sum_j E^j,
    non-decreasing, <= OPT."""
    for seed in range(60):
        p = synth.random_ilp(500 + seed, n=10, m=7, kmax=6, coef=3)
        opt = bf.solve_exhaustive(p)
        o = oracle_mod.Oracle(p)
        prev = o.lower_bound()
        for t in range(10):
            o.pass_seq(t % 2 == 0, 0.5)
            lam = o.lam()
            assert _feasibility(p, lam) <= 1e-9 * (1 + np.abs(p.cost).max())
            assert np.all(o.deferred() == 0.0)
            lb = o.lower_bound()
            assert abs(lb - _raw_bound(p, lam)) <= 1e-9 * (1 + abs(lb))
            assert lb >= prev - 1e-9 * (1 + abs(lb)), (seed, t)
            if opt is not None:  # (some random programs are jointly infeasible)
                assert lb <= opt + 1e-9 * (1 + abs(opt))
            prev = lb


def test_seq_lap_reaches_assignment_optimum(oracle_mod):
    """LAP special case (Birkhoff): the sequential scheme also closes the gap on
    the literal 4x4 matrix (OPT = 10)."""
    p = synth.lap(synth.LAP4_LITERAL)
    o = oracle_mod.Oracle(p)
    assert o.lower_bound() == 6.5
    o.iterate_seq(50, 0.5)
    assert abs(o.lower_bound() - 10.0) <= 1e-6


def test_seq_needs_no_pending_deferred_term(oracle_mod):
    """A pending deferred correction (after a deferred pass) must be finalized
    first; finalize -> sequential -> deferred passes compose."""
    p = synth.spec_two_constraint()
    o = oracle_mod.Oracle(p)
    o.pass_(True, 0.5)
    with pytest.raises(oracle_mod.OracleError) as e:
        o.pass_seq(True, 0.5)
    assert e.value.code == 6
    o.finalize()
    o.pass_seq(True, 0.5)
    o.pass_(False, 0.5)  # deferred pass after a sequential one: avg = 0
    assert o.lower_bound() <= bf.solve_exhaustive(p) + 1e-9
