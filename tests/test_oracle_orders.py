"""Pins of the oracle's from-definition distance recomputation (oracle.c
forward_dp / backward_dp) and of the state-setting entry points, -m "not gpu".

The incremental reuse of P:315-316 only holds while passes alternate; every
other call sequence -- a backward pass first, two passes in the same
direction, a pass after finalize, after set_lambda or after a primal
perturbation -- makes the oracle recompute shp(r, .) (forward_dp, P:319-324
with reading A4) or shp(., T) (backward_dp) from the current
lambda.  Each check below compares every recorded min-marginal of such a pass
with brute-force Eq. (MM) P:611 over the enumerated X_j (tests/bruteforce.py)
at the lambda the paper's order makes current at visit time (A3), so a
wrong arc, index or sign in either DP fails here.  The raw dual energy
(oracle_dual_energy) and the bound after oracle_set_lambda are checked
against sum_j E^j by enumeration plus the free-variable term (A13)
and the outstanding deferred term of the lifted bound (A7).
"""
import numpy as np
import pytest

import synth
from tests import bruteforce as bf


def _slots(problem):
    return [(j, h) for j in range(problem.n_cons) for h in range(int(problem.row_ptr[j + 1] - problem.row_ptr[j]))]


def _feasible_sets(problem):
    return [bf.feasible_set(problem.row(j)[1], problem.row(j)[2], problem.row(j)[3]) for j in range(problem.n_cons)]


def _free_term(problem):
    used = np.zeros(problem.n_vars, bool)
    used[problem.col_var] = True
    return float(np.minimum(problem.cost[~used], 0.0).sum())


def _check_pass(o, problem, X, fwd, omega):
    """One oracle pass; every recorded (m0, m1) == brute-force Eq. (MM) at the
    visit-time lambda (hops already visited in this pass updated, the others not)."""
    lam_pre = o.lam().copy()
    o.pass_(fwd, omega)
    lam_post = o.lam()
    m0, m1 = o.min_marginals()
    starts = problem.row_ptr
    for s, (j, h) in enumerate(_slots(problem)):
        a, b = int(starts[j]), int(starts[j + 1])
        k = b - a
        before = np.arange(k) < h if fwd else np.arange(k) > h
        seen = np.where(before, lam_post[a:b], lam_pre[a:b])
        e0, e1 = bf.min_marginal(X[j], seen, h)
        assert m0[s] == pytest.approx(e0, abs=1e-9), (fwd, j, h)
        assert m1[s] == pytest.approx(e1, abs=1e-9), (fwd, j, h)


def _energy_sum(problem, X, lam):
    starts = problem.row_ptr
    return sum(bf.energy(X[j], lam[int(starts[j]):int(starts[j + 1])]) for j in range(problem.n_cons)) \
        + _free_term(problem)


# direction sequences that break the alternation at every possible place
ORDERS = [
    "B",          # create -> backward (forward_dp from the initial lambda)
    "BB",         # backward -> backward
    "FF",         # forward -> forward (backward_dp)
    "BFFBB",
    "FBBFFB",
    "BBFB",
]


@pytest.mark.parametrize("order", ORDERS)
def test_non_alternating_orders_vs_bruteforce(oracle_mod, order):
    for seed in range(25):
        p = synth.random_ilp(7000 + seed, n=8, m=4, kmax=6)
        o = oracle_mod.Oracle(p)
        X = _feasible_sets(p)
        for c in order:
            _check_pass(o, p, X, c == "F", 0.5)


def test_pass_after_finalize_vs_bruteforce(oracle_mod):
    """finalize recomputes both distance directions; either pass after it."""
    for seed in range(20):
        p = synth.random_ilp(7100 + seed, n=8, m=4, kmax=6)
        for first in (True, False):
            o = oracle_mod.Oracle(p)
            X = _feasible_sets(p)
            o.iterate(2, 0.5)
            o.pass_(True, 0.5)
            o.finalize(averaged=bool(seed % 2))
            _check_pass(o, p, X, first, 0.5)
            _check_pass(o, p, X, not first, 0.5)


def test_set_lambda_then_passes_vs_bruteforce(oracle_mod):
    """oracle_set_lambda with an arbitrary lambda: the bound is sum_j E^j(lambda)
    (+ free term, + the outstanding min(delta_bar, 0) of A7), and the next pass
    in either direction sees distances recomputed from that lambda."""
    rng = np.random.default_rng(11)
    for seed in range(20):
        p = synth.random_ilp(7200 + seed, n=8, m=4, kmax=6)
        X = _feasible_sets(p)
        for fwd in (True, False):
            o = oracle_mod.Oracle(p)
            lam = rng.uniform(-3, 3, o.num_slots())
            o.set_lambda(lam)
            assert np.array_equal(o.lam(), lam)
            want = _energy_sum(p, X, lam)
            assert o.dual_energy() == pytest.approx(want, abs=1e-12)
            assert o.lower_bound() == pytest.approx(want, abs=1e-12)   # delta_bar = 0 here
            _check_pass(o, p, X, fwd, 0.5)
            _check_pass(o, p, X, fwd, 0.5)   # same direction again: recompute after a pass


def test_set_lambda_mid_run_keeps_deferred_term(oracle_mod):
    """set_lambda after a pass: delta_bar is untouched, so the lifted bound (A7)
    is sum_j E^j(lambda) + sum min(delta_bar, 0) + free term."""
    rng = np.random.default_rng(5)
    for seed in range(15):
        p = synth.random_ilp(7300 + seed, n=8, m=4, kmax=6)
        X = _feasible_sets(p)
        o = oracle_mod.Oracle(p)
        o.iterate(1, 0.5)
        o.pass_(True, 0.5)
        dbar = o.deferred().copy()
        lam = o.lam() + rng.uniform(-1, 1, o.num_slots())
        o.set_lambda(lam)
        assert np.array_equal(o.deferred(), dbar)
        want = _energy_sum(p, X, lam)
        assert o.dual_energy() == pytest.approx(want, abs=1e-12)
        assert o.lower_bound() == pytest.approx(want + float(np.minimum(dbar, 0).sum()), abs=1e-12)
        _check_pass(o, p, X, False, 0.5)


def test_dual_energy_during_run_vs_bruteforce(oracle_mod):
    """oracle_dual_energy == sum_j E^j(lambda^j) by enumeration + free term, at
    every point of a run, and lower_bound == it + sum min(delta_bar, 0) (A7)."""
    for seed in range(20):
        p = synth.random_ilp(7400 + seed, n=9, m=5, kmax=6)
        X = _feasible_sets(p)
        o = oracle_mod.Oracle(p)
        for t in range(6):
            o.pass_(t % 2 == 0, 0.5)
            lam = o.lam()
            want = _energy_sum(p, X, lam)
            assert o.dual_energy() == pytest.approx(want, abs=1e-9)
            assert o.lower_bound() == pytest.approx(want + float(np.minimum(o.deferred(), 0).sum()), abs=1e-9)


def test_pass_after_primal_perturbation_vs_bruteforce(oracle_mod):
    """A primal perturbation changes lambda outside a pass; the next
    pass (either direction) recomputes its distances from the perturbed lambda."""
    hit = 0
    for seed in range(40):
        p = synth.random_ilp(7500 + seed, n=8, m=4, kmax=6)
        X = _feasible_sets(p)
        for fwd in (True, False):
            o = oracle_mod.Oracle(p)
            o.iterate(2, 0.5)
            lam0 = o.lam().copy()
            und, _ = o.primal_step(0, 0.7, seed=seed)
            if und == 0:
                continue
            assert not np.array_equal(o.lam(), lam0)
            hit += 1
            _check_pass(o, p, X, fwd, 0.5)
    assert hit >= 10
