"""GPU primal rounding (Alg. 2, §8 row f1) vs the oracle's.

* one classification + perturbation step from a state that is bit-identical on
  both sides (LAP literal, dyadic iterations): same undecided count, same
  labeling, same perturbed lambda (same counter-based r, fp64);
* the full loop returns labelings that satisfy every row, with objective >=
  brute-force OPT >= the dual bound; the dual state is restored afterwards.
"""
import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth
from tests import bruteforce as bf

pytestmark = pytest.mark.gpu


def _feasible(p, x):
    for j in range(p.n_cons):
        v, c, rel, rhs = p.row(j)
        if not bf.row_sat(int(np.dot(x[v].astype(np.int64), c.astype(np.int64))), rel, rhs):
            return False
    return True


@pytest.mark.parametrize("iters", [1, 2])
def test_primal_step_bit_exact_lap(oracle_mod, iters):
    p = synth.lap(synth.LAP4_LITERAL)
    o = oracle_mod.Oracle(p)
    g = F.Solver(p, precision=64)
    o.iterate(iters, 0.5); g.iterate(iters, 0.5)
    assert np.array_equal(g.lam(), o.lam()) and np.array_equal(g.deferred(), o.deferred())
    for rnd, delta in ((0, 1.0), (1, 1.2), (2, 1.44)):
        uo, xo = o.primal_step(rnd, delta, seed=7)
        ug, xg = g.primal_step(rnd, delta, seed=7)
        assert uo == ug and np.array_equal(xo, xg)
        assert np.array_equal(g.lam(), o.lam())
        o.iterate(1, 0.5); g.iterate(1, 0.5)


def test_round_primal_random(oracle_mod):
    ok = tried = 0
    for seed in range(40):
        p = synth.random_ilp(5000 + seed, n=10, m=6, kmax=5)
        opt = bf.solve_exhaustive(p)
        if opt is None:
            continue
        tried += 1
        g = F.Solver(p, precision=64)
        g.iterate(20, 0.5)
        lb, lam = g.lower_bound(), g.lam()
        try:
            x, rounds, obj = g.round_primal(seed=seed)
        except F.FastdogError as e:
            assert e.code == 8
            continue
        assert _feasible(p, x)
        assert obj == pytest.approx(float(p.cost @ x)) and obj >= opt - 1e-9 >= lb - 2e-9
        assert np.array_equal(g.lam(), lam) and g.lower_bound() == lb  # state restored
        ok += 1
    assert tried >= 20 and ok >= 0.9 * tried, (ok, tried)


@pytest.mark.parametrize("mode", ["", "rc", "tma"])
def test_round_primal_workloads(oracle_mod, monkeypatch, mode):
    """Every sweep design (default choice, recompute, TMA store) under the
    rounding loop's snapshot / perturb / iterate / restore sequence."""
    if mode:
        monkeypatch.setenv("FDOG_SWEEP", mode)
    for p in (synth.gm_worms_like(14, n_src=40, k_cand=4, knn=4), synth.mrf_potts(14, H=6, W=7, L=3),
              synth.lap(synth.LAP4_LITERAL)):
        g = F.Solver(p, precision=32)
        g.iterate(30, 0.5)
        lb = g.lower_bound()
        lam = g.lam()
        x, rounds, obj = g.round_primal(seed=1, max_rounds=200)
        assert _feasible(p, x) and obj >= lb - 1e-3 * max(1.0, abs(lb))
        assert np.array_equal(g.lam(), lam) and g.lower_bound() == lb  # state restored
        g.iterate(2, 0.5)  # and the solver continues from it
        assert g.lower_bound() >= lb - 1e-5 * max(1.0, abs(lb))


def test_round_primal_restores_min_marginals():
    """keep_state = 0 restores the recorded min-marginals too (record_mm), so
    fdog_min_marginals after the rounding returns those of the restored last pass."""
    p = synth.gm_worms_like(15, n_src=30, k_cand=4, knn=4)
    g = F.Solver(p, precision=64, record_mm=True)
    g.iterate(10, 0.5)
    m0, m1 = g.min_marginals()
    try:
        g.round_primal(seed=3, max_rounds=200)
    except F.FastdogError as e:   # no consensus: the state is restored all the same
        assert e.code == 8
    a0, a1 = g.min_marginals()
    assert np.array_equal(a0, m0) and np.array_equal(a1, m1)
