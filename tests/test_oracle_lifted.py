"""Pins of the oracle's lifted representation (oracle_set_lifted; P:32-57,
reading A8) against what the paper and brute force fix
(-m "not gpu"): the enumeration implementation in tests/bruteforce.py
(lifted_passes: no BDDs, no shortest paths), the original-space update it must
reproduce (P:46-49 vs P:641), and Prop. 1 on instances with forced variables."""
import numpy as np
import pytest

import synth
from tests import bruteforce as bf

DIRS = [True, False, True, False, False, True, True, False]


def _lifted(oracle_mod, p):
    o = oracle_mod.Oracle(p)
    o.set_lifted()
    return o


@pytest.mark.parametrize("seed", range(30))
def test_lifted_passes_equal_enumeration(oracle_mod, seed):
    """Every pass (including non-alternating orders): lambda^{j,0}, lambda^{j,1},
    delta_bar and the bound equal the enumeration at 1e-9; instances with
    forced variables (clamped sides, A5) in every third seed."""
    p = synth.random_ilp(3100 + seed, n=9, m=6, kmax=6, coef=3, forced_ok=seed % 3 == 0)
    o = _lifted(oracle_mod, p)
    s = max(1.0, float(np.abs(p.cost).max()))
    for t, (e0, e1, elb, edb) in enumerate(bf.lifted_passes(p, DIRS)):
        o.pass_(DIRS[t], 0.5)
        l0, l1 = o.lifted()
        C = oracle_mod.default_clamp(p.cost)
        tol = 1e-9 * max(s, C * 0.5 if seed % 3 == 0 else s)
        assert np.max(np.abs(l0 - e0), initial=0) <= tol, f"pass {t} lambda0"
        assert np.max(np.abs(l1 - e1), initial=0) <= tol, f"pass {t} lambda1"
        assert np.max(np.abs(o.deferred() - edb), initial=0) <= tol
        assert abs(o.lower_bound() - elb) <= 1e-9 * (abs(elb) + s), f"pass {t} bound"


@pytest.mark.parametrize("seed", range(20))
def test_lifted_reproduces_original_space(oracle_mod, seed):
    """lambda^1 - lambda^0 follows the original-space update (P:46-49 vs P:641)
    and, without forced variables, the lifted bound equals the bound of
    reading A7 (sum_j E^j + sum min(delta_bar, 0)) of the plain oracle."""
    p = synth.random_ilp(3300 + seed, n=10, m=6, kmax=6, coef=3)
    o = _lifted(oracle_mod, p)
    r = oracle_mod.Oracle(p)
    s = max(1.0, float(np.abs(p.cost).max()))
    for fwd in DIRS:
        o.pass_(fwd, 0.5)
        r.pass_(fwd, 0.5)
        assert np.max(np.abs(o.lam() - r.lam())) <= 1e-9 * s
        assert abs(o.lower_bound() - r.lower_bound()) <= 1e-9 * (abs(r.lower_bound()) + s)


@pytest.mark.parametrize("seed", range(25))
def test_lifted_bound_forced_variables(oracle_mod, seed):
    """Prop. 1 with forced variables: the lifted bound is a plain sum of per-BDD
    shortest paths, <= the brute-force optimum and non-decreasing
     at 1e-9 -- no clamp-sized cancellation (the single-sided bound
    carries +-C terms that cancel only up to C eps, A5)."""
    for t in range(50):  # the first globally feasible instance of this seed
        p = synth.random_ilp(3500 + 97 * seed + t, n=9, m=6, kmax=6, coef=3, forced_ok=True)
        opt = bf.solve_exhaustive(p)
        if opt is not None:
            break
    o = _lifted(oracle_mod, p)
    lbs = [o.lower_bound()]
    for _ in range(15):
        o.iterate(1, 0.5)
        lbs.append(o.lower_bound())
    lbs = np.array(lbs)
    assert np.all(lbs <= opt + 1e-9 * (1 + abs(opt)))
    assert np.all(np.diff(lbs) >= -1e-9 * (1 + np.abs(lbs[:-1])))


def test_lifted_finalize_feasible(oracle_mod):
    """Final correction in lifted form: lambda^{j,b} += max(+-delta_bar,
    0); afterwards sum_j (lambda^1 - lambda^0)_i = c_i (I5) and the bound is
    sum_j E^j of the original-space lambda."""
    for seed in range(10):
        p = synth.random_ilp(3700 + seed, n=10, m=7, kmax=6, coef=3, forced_ok=seed % 2 == 0)
        o = _lifted(oracle_mod, p)
        o.iterate(5, 0.5)
        o.finalize()
        lam = o.lam()
        sums = np.zeros(p.n_vars)
        np.add.at(sums, p.col_var, lam)
        deg = np.bincount(p.col_var, minlength=p.n_vars)
        C = oracle_mod.default_clamp(p.cost)
        assert np.allclose(sums[deg > 0], p.cost[deg > 0], atol=1e-9 * C)
        assert np.allclose(o.deferred(), 0.0)


def test_lifted_state_rules(oracle_mod):
    p = synth.spec_two_constraint()
    o = oracle_mod.Oracle(p)
    o.pass_(True, 0.5)
    with pytest.raises(oracle_mod.OracleError):
        o.set_lifted()  # only before the first pass
    o = _lifted(oracle_mod, p)
    o.pass_(True, 0.5)
    for call in (lambda: o.pass_seq(True, 0.5), lambda: o.finalize(averaged=True), lambda: o.dual_energy()):
        with pytest.raises(oracle_mod.OracleError):
            call()
