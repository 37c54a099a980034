"""Pins of the oracle's Alg. "Perturbation Primal Rounding" (§8 row f1).

Independent references: brute-force optimum (Eq. BP), constraint
checks, the paper's per-branch update rules checked on min-marginals the test
recomputes by brute force (Eq. MM), and SPEC's examples.
The random draw r of P:206 is the counter-based generator splitmix64(seed,
round, i) both sides implement; the test re-derives r from it.
"""
import numpy as np
import pytest

import synth
from tests import bruteforce as bf

MASK = (1 << 64) - 1


def _uniform(seed, rnd, i):
    z = (seed * 0x9E3779B97F4A7C15 + rnd * 0xBF58476D1CE4E5B9 + i * 0x94D049BB133111EB + 1) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    z ^= z >> 31
    return (z >> 11) * (1.0 / 9007199254740992.0)


def _feasible(p, x):
    for j in range(p.n_cons):
        v, c, rel, rhs = p.row(j)
        if not bf.row_sat(int(np.dot(x[v].astype(np.int64), c.astype(np.int64))), rel, rhs):
            return False
    return True


def test_min_x_plus_y(oracle_mod):
    """{min x+y; x+y>=1}: the dual fixed point ties (m1 = m0); rounding breaks the
    tie (reading R1) and returns an optimal labeling of cost 1."""
    p = synth.from_rows(2, [1.0, 1.0], [([0, 1], [1, 1], 1, 1)])
    o = oracle_mod.Oracle(p)
    o.iterate(5, 0.5)
    x, rounds = o.round_primal(seed=3)
    assert _feasible(p, x) and float(p.cost @ x) == 1.0 and rounds >= 1


def test_no_constraints(oracle_mod):
    """No constraints, c = (-2, 3): x = (1, 0), zero rounds."""
    p = synth.from_rows(2, [-2.0, 3.0], [])
    o = oracle_mod.Oracle(p)
    x, rounds = o.round_primal()
    assert list(x) == [1, 0] and rounds == 0


def test_lap_literal_optimal(oracle_mod):
    """LAP literal: the dual reaches OPT = 10 (Birkhoff) and the min-marginals
    agree, so rounding reads off an optimal assignment without perturbation."""
    cm = synth.LAP4_LITERAL
    p = synth.lap(cm)
    o = oracle_mod.Oracle(p)
    o.iterate(50, 0.5)
    x, rounds = o.round_primal()
    assert _feasible(p, x)
    assert float(p.cost @ x) == bf.assignment_opt(cm) == 10.0
    assert rounds == 0


def test_step_follows_the_four_branches(oracle_mod):
    """One step of Alg. 2 on a random state: per variable, lambda moves by +delta
    (all m1 > m0), -delta (all m1 < m0), r*delta (all
    equal) or sign(d_i)*|r|*delta (else), applied to the
    min-marginals recorded in the last pass (those are pinned against brute
    force in test_oracle.py::test_incremental_min_marginals_random)."""
    checked = 0
    for seed in range(15):
        p = synth.random_ilp(3000 + seed, n=8, m=5, kmax=5)
        o = oracle_mod.Oracle(p)
        o.iterate(2, 0.5)
        o.pass_(True, 0.5)       # min-marginals of a forward pass, recorded per slot
        m0, m1 = o.min_marginals()
        lam0 = o.lam().copy()
        delta, rnd, rseed = 1.7, 4, 11
        nc, x = o.primal_step(rnd, delta, rseed)
        lam1 = o.lam()
        var_of = p.col_var
        expect_nc = 0
        for i in range(p.n_vars):
            sl = np.flatnonzero(var_of == i)
            if sl.size == 0:
                continue
            d = m1[sl] - m0[sl]
            sg = np.sign(d)
            pos, neg, zero = (sg > 0).all(), (sg < 0).all(), (sg == 0).all()
            assert x[i] == int(neg)
            if not (pos or neg):      # reading R1: ties are undecided too
                expect_nc += 1
        assert nc == expect_nc
        if nc == 0:
            assert np.array_equal(lam1, lam0)
            continue
        for i in range(p.n_vars):
            sl = np.flatnonzero(var_of == i)
            if sl.size == 0:
                continue
            d = m1[sl] - m0[sl]
            sg = np.sign(d)
            r = delta * (2.0 * _uniform(rseed, rnd, i) - 1.0)
            if (sg > 0).all():
                step = delta
            elif (sg < 0).all():
                step = -delta
            elif (sg == 0).all():
                step = r * delta
            else:
                step = np.sign(d.sum()) * abs(r) * delta
            assert np.allclose(lam1[sl] - lam0[sl], step, atol=1e-12)
        checked += 1
    assert checked >= 5


def test_random_instances_feasible_and_bounded(oracle_mod):
    """SPEC acceptance 7 / weak duality: rounding returns a feasible labeling on
    >= 95% of random feasible instances; its objective is >= OPT >= LB."""
    ok = tried = 0
    for seed in range(100):
        p = synth.random_ilp(4000 + seed, n=10, m=6, kmax=5)
        opt = bf.solve_exhaustive(p)
        if opt is None:
            continue
        tried += 1
        o = oracle_mod.Oracle(p)
        o.iterate(20, 0.5)
        lb = o.lower_bound()
        try:
            x, _ = o.round_primal(seed=seed)
        except oracle_mod.OracleError as e:
            assert e.code == 7
            continue
        if not _feasible(p, x):
            continue
        obj = float(p.cost @ x)
        assert obj >= opt - 1e-9 >= lb - 2e-9
        ok += 1
    assert tried >= 50 and ok >= 0.95 * tried, (ok, tried)


def test_determinism(oracle_mod):
    p = synth.gm_worms_like(3, n_src=20, k_cand=3, knn=3)
    a = oracle_mod.Oracle(p, n_threads=1)
    b = oracle_mod.Oracle(p, n_threads=4)
    a.iterate(10, 0.5); b.iterate(10, 0.5)
    xa, ra = a.round_primal(seed=5)
    xb, rb = b.round_primal(seed=5)
    assert ra == rb and np.array_equal(xa, xb)
