"""Lifted two-sided storage on the GPU (fdog_options::lifted, SURVEY §8 f3;
P:32-57, reading A8) against the oracle's lifted representation (pinned in
tests/test_oracle_lifted.py against an enumeration implementation): fp64,
every pass, lambda^{j,0} and lambda^{j,1} per slot and the bound at 1e-9 --
including instances with forced variables, where the bound is the plain sum
of per-BDD shortest paths (no clamp-sized terms)."""
import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth

pytestmark = pytest.mark.gpu

DIRS = [True, False, True, False, False, True, True, False, True, False]


def _pair(oracle_mod, p, precision=64, record_mm=True):
    o = oracle_mod.Oracle(p)
    o.set_lifted()
    g = F.Solver(p, precision=precision, record_mm=record_mm, lifted=True)
    return g, o


def _check(g, o, p, tol, what):
    s = max(1.0, float(np.abs(p.cost).max()))
    a0, a1 = g.lifted()
    b0, b1 = o.lifted()
    assert np.max(np.abs(a0 - b0), initial=0) <= tol * s, f"{what}: lambda0"
    assert np.max(np.abs(a1 - b1), initial=0) <= tol * s, f"{what}: lambda1"
    assert np.max(np.abs(g.lam() - o.lam()), initial=0) <= tol * s, f"{what}: lambda1 - lambda0"
    assert np.max(np.abs(g.deferred() - o.deferred()), initial=0) <= tol * s, f"{what}: delta_bar"
    assert abs(g.lower_bound() - o.lower_bound()) <= tol * (abs(o.lower_bound()) + s), f"{what}: bound"


@pytest.mark.parametrize("name,make", [
    ("random_forced", lambda: synth.random_ilp(41, n=30, m=40, kmax=8, coef=4, forced_ok=True)),
    ("random_wide", lambda: synth.random_ilp(42, n=40, m=60, kmax=12, coef=5)),
    ("gm", lambda: synth.gm_worms_like(43, n_src=60, k_cand=6, knn=6)),
    ("mrf", lambda: synth.mrf_potts(43, H=10, W=12, L=4)),
    ("gap", lambda: synth.gap(43, jobs=40, agents=5)),
])
def test_lifted_matches_oracle(oracle_mod, name, make):
    p = make()
    g, o = _pair(oracle_mod, p)
    _check(g, o, p, 1e-12, "create")
    for t, fwd in enumerate(DIRS):
        g.pass_(fwd, 0.5)
        o.pass_(fwd, 0.5)
        _check(g, o, p, 1e-9, f"pass {t}")
        gm0, gm1 = g.min_marginals()
        om0, om1 = o.min_marginals()
        fin = np.isfinite(om0)
        assert np.array_equal(fin, np.isfinite(gm0))
        assert np.allclose(gm0[fin], om0[fin], rtol=1e-9, atol=1e-9 * max(1.0, float(np.abs(p.cost).max())))
    g.iterate(5, 0.5)
    o.iterate(5, 0.5)
    _check(g, o, p, 1e-8, "iterate")
    g.finalize()
    o.finalize()
    _check(g, o, p, 1e-8, "finalize")


def test_lifted_forced_bound_is_plain_sum(oracle_mod):
    """Forced variables: the single-sided bound carries +-C terms (A5) that
    cancel to C eps; the lifted bound does not.  fp32 and fp64 lifted bounds
    stay within 1e-4 relative of the oracle's lifted bound after 50
    iterations, monotone (Prop. 1)."""
    p = synth.random_ilp(44, n=30, m=40, kmax=8, coef=4, forced_ok=True)
    o = oracle_mod.Oracle(p)
    o.set_lifted()
    lbs = {}
    for prec in (64, 32):
        g = F.Solver(p, precision=prec, lifted=True)
        seq = [g.lower_bound()]
        for _ in range(10):
            g.iterate(5, 0.5)
            seq.append(g.lower_bound())
        lbs[prec] = np.array(seq)
    o.iterate(50, 0.5)
    ref = o.lower_bound()
    for prec, seq in lbs.items():
        assert abs(seq[-1] - ref) <= 1e-4 * max(1.0, abs(ref)), prec
        assert np.all(np.diff(seq) >= -1e-6 * (1 + np.abs(seq[:-1]))), prec


def test_lifted_state_rules():
    p = synth.spec_two_constraint()
    g = F.Solver(p, precision=64, lifted=True)
    g.iterate(1, 0.5)
    for call in (lambda: g.pass_seq(True, 0.5), lambda: g.finalize(averaged=True),
                 lambda: g.set_state(g.lam(), g.deferred())):
        with pytest.raises(F.FastdogError) as e:
            call()
        assert e.value.code == 6
    h = F.Solver(p, precision=64)
    with pytest.raises(F.FastdogError) as e:
        h.lifted()
    assert e.value.code == 6
    plan = F.Plan(p, precision=64)
    with pytest.raises(F.FastdogError) as e:
        F.Solver(plan=plan, precision=64, lifted=True)  # plan packed without the option
    assert e.value.code == 1
