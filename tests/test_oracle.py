"""Pins of the fp64 oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins.  Independent references used here:
brute-force enumeration (tests/bruteforce.py), closed forms, the paper's
worked example (tests/golden/figure_bdd.json), the survey's independently
computed trajectories (tests/golden/survey_derived.json), and an
enumeration-based implementation of the appendix's *lifted* representation
(reading A8), which shares no code or mechanism with the oracle's
BDD shortest paths.
"""
import json
import os

import numpy as np
import pytest

import synth
from tests import bruteforce as bf

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _slot_of(problem):
    """canonical slot -> (j, h); slots are (j asc, h asc)."""
    out = []
    for j in range(problem.n_cons):
        k = int(problem.row_ptr[j + 1] - problem.row_ptr[j])
        out += [(j, h) for h in range(k)]
    return out


def _paths(vars_, hs, lo, hi):
    """Enumerate root->top paths of a BDD (Def. P:259-270)."""
    k = len(vars_)
    out = []

    def rec(v, h, bits):
        if h == k:
            return
        for beta, w in ((0, lo[v]), (1, hi[v])):
            if w == -1:
                continue
            if h == k - 1:
                if w == -2:
                    out.append(tuple(bits + [beta]))
                continue
            assert hs[h + 1] <= w < hs[h + 2], "arc must go to the next partition (P:253-254)"
            rec(w, h + 1, bits + [beta])

    rec(0, 0, [])
    return out


# ---------------------------------------------------------------- BDD compile

def test_figure_partition_sizes(oracle_mod):
    g = _gold("figure_bdd.json")
    o = oracle_mod.Oracle(synth.figure_bdd_problem())
    assert list(o.hop_widths(0)) == g["partition_sizes"]
    vars_, hs, lo, hi = o.bdd(0)
    got = sorted("".join(map(str, p)) for p in _paths(vars_, hs, lo, hi))
    assert got == sorted(g["feasible_set"])
    # some node of P_3 has s^0 in P_4 and s^1 = bottom (c2)
    p3 = range(hs[2], hs[3])
    assert any(hs[3] <= lo[v] < hs[4] and hi[v] == -1 for v in p3)


def test_random_rows_path_sets(oracle_mod):
    """Paths == brute-force X_j on 500 random rows."""
    rng = np.random.default_rng(123)
    done = 0
    while done < 500:
        k = int(rng.integers(1, 11))
        a = rng.integers(-5, 6, size=k)
        a[a == 0] = 1
        rel = int(rng.choice([-1, 0, 1]))
        b = int(rng.integers(-6, 7))
        X = bf.feasible_set(a, rel, b)
        p = synth.from_rows(k, np.zeros(k), [(np.arange(k), a, rel, b)])
        if X.shape[0] == 0:
            with pytest.raises(oracle_mod.OracleError) as e:
                oracle_mod.Oracle(p)
            assert e.value.code == 2
            continue
        o = oracle_mod.Oracle(p)
        vars_, hs, lo, hi = o.bdd(0)
        paths = _paths(vars_, hs, lo, hi)
        assert len(paths) == len(set(paths))
        assert set(paths) == set(map(tuple, X.tolist()))
        # canonical: no two nodes in a partition with equal successor pairs
        for h in range(k):
            sig = [(lo[v], hi[v]) for v in range(hs[h], hs[h + 1])]
            assert len(sig) == len(set(sig))
            assert all(s != (-1, -1) for s in sig)
        assert hs[1] - hs[0] == 1  # P_1 = {r}
        done += 1


@pytest.mark.parametrize("k", [1, 2, 3, 5, 11, 40])
def test_closed_form_node_counts(oracle_mod, k):
    """one-hot(k) = at-most-one(k) = 2k-1; sum y - x = 0 over k vars = 2k-1."""
    n = k
    for rel, rhs in ((0, 1), (-1, 1)):
        o = oracle_mod.Oracle(synth.from_rows(n, np.zeros(n), [(np.arange(n), np.ones(n), rel, rhs)]))
        assert o.total_nodes() == max(2 * k - 1, 1)
    if k >= 2:
        c = np.ones(k); c[0] = -1   # x first
        o = oracle_mod.Oracle(synth.from_rows(k, np.zeros(k), [(np.arange(k), c, 0, 0)]))
        assert o.total_nodes() == 2 * k - 1
        c = np.ones(k); c[-1] = -1  # x last
        o = oracle_mod.Oracle(synth.from_rows(k, np.zeros(k), [(np.arange(k), c, 0, 0)]))
        assert o.total_nodes() == 2 * k - 1


def test_potts_cut_row(oracle_mod):
    """x_il - x_jl - z_e <= 0 over 3 variables: 5 nodes."""
    o = oracle_mod.Oracle(synth.from_rows(3, np.zeros(3), [([0, 1, 2], [1, -1, -1], -1, 0)]))
    assert o.total_nodes() == 5


def test_trivial_rows(oracle_mod):
    o = oracle_mod.Oracle(synth.from_rows(1, [1.0], [([0], [1], -1, 1)]))       # x <= 1
    _, hs, lo, hi = o.bdd(0)
    assert list(hs) == [0, 1] and lo[0] == -2 and hi[0] == -2
    with pytest.raises(oracle_mod.OracleError) as e:                            # x+y <= -1
        oracle_mod.Oracle(synth.from_rows(2, [0, 0], [([0, 1], [1, 1], -1, -1)]))
    assert e.value.code == 2


# ---------------------------------------------------------------- min-marginals

def test_figure_min_marginals(oracle_mod):
    """Worked example P:303 with lambda = (2,3,1,4): MMs by Eq. (MM), E = 0."""
    g = _gold("figure_bdd.json")
    X = bf.feasible_set(g["coef"], g["rel"], g["rhs"])
    for h, name in enumerate("abcd"):
        assert bf.min_marginal(X, g["lambda"], h) == tuple(g["min_marginals"][name])
    assert bf.energy(X, g["lambda"]) == g["energy"]
    # the oracle starts from lambda = c/|J_i| = c here; its first forward visit of
    # hop a sees exactly the figure's lambda
    o = oracle_mod.Oracle(synth.figure_bdd_problem())
    assert o.lower_bound() == 0.0
    o.pass_(True, 0.5)
    m0, m1 = o.min_marginals()
    assert (m0[0], m1[0]) == tuple(g["min_marginals"]["a"])


def _run_with_visit_checks(oracle_mod, problem, n_iter, omega):
    """Run passes; after each, check every recorded MM against brute force at the
    lambda the paper's order says was current at visit time (A3)."""
    o = oracle_mod.Oracle(problem)
    slots = _slot_of(problem)
    X = [bf.feasible_set(problem.row(j)[1], problem.row(j)[2], problem.row(j)[3])
         for j in range(problem.n_cons)]
    starts = problem.row_ptr
    history = [o.lower_bound()]
    for t in range(2 * n_iter):
        fwd = t % 2 == 0
        lam_pre = o.lam().copy()
        o.pass_(fwd, omega)
        lam_post = o.lam()
        m0, m1 = o.min_marginals()
        for s, (j, h) in enumerate(slots):
            a, b = int(starts[j]), int(starts[j + 1])
            pre, post = lam_pre[a:b], lam_post[a:b]
            k = b - a
            seen = np.where(np.arange(k) < h, post, pre) if fwd else np.where(np.arange(k) > h, post, pre)
            e0, e1 = bf.min_marginal(X[j], seen, h)
            assert m0[s] == pytest.approx(e0, abs=1e-9) and m1[s] == pytest.approx(e1, abs=1e-9)
            # I4: min(m0, m1) = E^j(lambda at visit time)
            assert min(m0[s], m1[s]) == pytest.approx(bf.energy(X[j], seen), abs=1e-9)
        history.append(o.lower_bound())
    return o, history


def test_incremental_min_marginals_random(oracle_mod):
    """incremental MMs equal brute-force Eq. (MM) at every visit."""
    for seed in range(40):
        p = synth.random_ilp(seed, n=8, m=4, kmax=6)
        _run_with_visit_checks(oracle_mod, p, n_iter=5, omega=0.5)


# ---------------------------------------------------------------- Prop. 1 invariants

def _feasibility_residual(problem, lam, delta):
    """max_i |sum_{j in J_i} (lambda_i^j + delta_ij) - c_i|."""
    col = problem.col_var
    acc = np.zeros(problem.n_vars)
    np.add.at(acc, col, lam + delta)
    used = np.zeros(problem.n_vars, bool)
    used[col] = True
    return float(np.max(np.abs(acc - problem.cost)[used])) if used.any() else 0.0


@pytest.mark.parametrize("omega", [0.5, 0.3, 1.0])
def test_prop1_invariants_random(oracle_mod, omega):
    """I1 feasibility, I2 monotone LB, I3 LB <= OPT, I5."""
    checked = 0
    for seed in range(60):
        p = synth.random_ilp(1000 + seed, n=10, m=6, kmax=6)
        opt = bf.solve_exhaustive(p)
        if opt is None:
            continue
        o = oracle_mod.Oracle(p)
        lbs = [o.lower_bound()]
        assert _feasibility_residual(p, o.lam(), np.zeros(o.num_slots())) < 1e-12
        for t in range(30):
            o.pass_(t % 2 == 0, omega)
            assert _feasibility_residual(p, o.lam(), o.deferred()) < 1e-9
            lbs.append(o.lower_bound())
        lbs = np.array(lbs)
        assert np.all(np.diff(lbs) >= -1e-9 * (1 + np.abs(lbs[:-1])))
        assert lbs.max() <= opt + 1e-9
        o.finalize()
        assert _feasibility_residual(p, o.lam(), np.zeros(o.num_slots())) < 1e-9
        assert o.lower_bound() <= opt + 1e-9
        assert o.lower_bound() >= lbs[-1] - 1e-9   # finalized >= lifted
        checked += 1
    assert checked >= 40


def test_averaged_finalize_feasible(oracle_mod):
    """Averaged final correction (P:673 prose): sum_j lambda_i^j = c_i afterwards,
    and its bound is a valid lower bound (<= OPT)."""
    for seed in range(30):
        p = synth.random_ilp(6000 + seed, n=10, m=6, kmax=6)
        opt = bf.solve_exhaustive(p)
        if opt is None:
            continue
        o = oracle_mod.Oracle(p)
        o.iterate(4, 0.5)
        o.pass_(True, 0.5)
        o.finalize(averaged=True)
        assert _feasibility_residual(p, o.lam(), np.zeros(o.num_slots())) < 1e-9
        assert o.lower_bound() <= opt + 1e-9
        assert np.all(o.deferred() == 0)


def test_single_constraint_is_exact(oracle_mod):
    """m = 1: the dual is the subproblem itself, so LB = OPT from init and stays."""
    for seed in range(20):
        p = synth.random_ilp(500 + seed, n=7, m=1, kmax=7)
        opt = bf.solve_exhaustive(p)
        v, c, rel, rhs = p.row(0)
        free = sum(min(p.cost[i], 0.0) for i in range(p.n_vars) if i not in set(v.tolist()))
        o = oracle_mod.Oracle(p)
        assert o.lower_bound() == pytest.approx(opt, abs=1e-12)
        o.iterate(5, 0.5)
        assert o.lower_bound() == pytest.approx(opt, abs=1e-9)
        assert free == pytest.approx(o.lower_bound() - bf.energy(bf.feasible_set(c, rel, rhs),
                                                                 p.cost[v]), abs=1e-9)


def test_lifted_representation_cross_check(oracle_mod):
    """Independent enumeration implementation of the appendix's lifted
    representation (update P:53-56 read as A8).  Its lifted energy
    sum_j E(lambda^{j,1}, lambda^{j,0}) must equal the oracle's bound (A7) after
    every pass, and lambda^1 - lambda^0 the oracle's lambda."""
    omega = 0.5
    for seed in range(25):
        p = synth.random_ilp(2000 + seed, n=9, m=5, kmax=6)
        o = oracle_mod.Oracle(p)
        rows = [p.row(j) for j in range(p.n_cons)]
        X = [bf.feasible_set(c, r, b) for (_, c, r, b) in rows]
        deg = np.bincount(p.col_var, minlength=p.n_vars)
        l1 = [p.cost[v] / deg[v] for (v, _, _, _) in rows]     # lambda^{j,1} = c/|J_i|
        l0 = [np.zeros(len(v)) for (v, _, _, _) in rows]       # lambda^{j,0} = 0
        mbar = [np.zeros((len(v), 2)) for (v, _, _, _) in rows]
        free = sum(min(p.cost[i], 0.0) for i in range(p.n_vars) if deg[i] == 0)
        for t in range(12):
            fwd = t % 2 == 0
            # averaging terms (omega/|J_i|) sum_k max(mbar^b - mbar^{1-b}, 0), per beta
            avg = np.zeros((p.n_vars, 2))
            for j, (v, _, _, _) in enumerate(rows):
                for h, i in enumerate(v):
                    d = mbar[j][h, 1] - mbar[j][h, 0]
                    avg[i, 1] += omega * max(d, 0.0) / deg[i]
                    avg[i, 0] += omega * max(-d, 0.0) / deg[i]
            newm = []
            for j, (v, _, _, _) in enumerate(rows):
                k = len(v)
                mm = np.zeros((k, 2))
                for h in (range(k) if fwd else reversed(range(k))):
                    vals = X[j] @ l1[j] + (1 - X[j]) @ l0[j]
                    m = [vals[X[j][:, h] == beta].min() for beta in (0, 1)]
                    mm[h] = m
                    l1[j][h] += -omega * max(m[1] - m[0], 0.0) + avg[v[h], 1]
                    l0[j][h] += -omega * max(m[0] - m[1], 0.0) + avg[v[h], 0]
                newm.append(mm)
            mbar = newm
            o.pass_(fwd, omega)
            lifted = sum(float(np.min(X[j] @ l1[j] + (1 - X[j]) @ l0[j])) for j in range(len(rows)))
            assert o.lower_bound() == pytest.approx(lifted + free, abs=1e-9)
            assert np.allclose(o.lam(), np.concatenate([a - b for a, b in zip(l1, l0)]), atol=1e-9)


# ---------------------------------------------------------------- worked instances

def test_figure_alone_trajectory(oracle_mod):
    g = _gold("survey_derived.json")["figure_alone_omega_0.5"]
    o = oracle_mod.Oracle(synth.figure_bdd_problem())
    o.pass_(True, 0.5)
    m0, m1 = o.min_marginals()
    assert np.allclose(np.stack([m0, m1], 1), g["forward_pass_min_marginals"], atol=0)
    assert np.array_equal(o.lam(), g["lambda_after_forward"])
    o.pass_(False, 0.5)
    assert np.array_equal(o.lam(), g["lambda_after_iteration"])
    assert np.array_equal(o.deferred() / 0.5, g["delta_over_omega_after_iteration"])
    assert o.lower_bound() == g["lower_bound"]


def test_spec_two_constraint(oracle_mod):
    g = _gold("survey_derived.json")["spec_two_constraint_omega_0.5"]
    p = synth.spec_two_constraint()
    assert bf.solve_exhaustive(p) == g["opt"]
    o = oracle_mod.Oracle(p)
    assert o.lower_bound() == g["lb0"]
    assert np.array_equal(o.lam(), [2, 1.5, 0.5, 4, 1.5, 0.5])
    o.iterate(1, 0.5)
    assert o.lower_bound() == g["lb_iter1"]
    assert np.array_equal(o.lam(), g["lambda0_iter1"] + g["lambda1_iter1"])
    o.iterate(9, 0.5)
    assert o.lower_bound() == pytest.approx(g["lb_iter10"], abs=1e-9)
    o.iterate(200, 0.5)
    assert o.lower_bound() == pytest.approx(g["lb_limit"], abs=1e-6)
    assert o.lower_bound() <= g["opt"]


def test_min_x_plus_y(oracle_mod):
    """{min x+y; x+y>=1}: lambda=(1,1), LB = 1 = OPT, a fixed point."""
    p = synth.from_rows(2, [1.0, 1.0], [([0, 1], [1, 1], 1, 1)])
    o = oracle_mod.Oracle(p)
    assert o.lower_bound() == 1.0 and list(o.lam()) == [1.0, 1.0]
    o.iterate(3, 0.5)
    assert o.lower_bound() == 1.0


def test_zero_iterations_untouched(oracle_mod):
    """omega anything, zero iterations -> multipliers untouched."""
    p = synth.spec_two_constraint()
    o = oracle_mod.Oracle(p)
    l0 = o.lam().copy()
    o.iterate(0, 0.7)
    assert np.array_equal(o.lam(), l0)


def test_lap4_literal(oracle_mod):
    """LB_0 by closed form, the survey's trajectory, LB_50 = OPT (Birkhoff)."""
    g = _gold("survey_derived.json")["lap4_literal_omega_0.5"]
    cm = np.array(g["cost"], dtype=float)
    p = synth.lap(cm)
    closed = 0.5 * (cm.min(axis=1).sum() + cm.min(axis=0).sum())
    opt = bf.assignment_opt(cm)
    assert opt == g["opt"] and bf.solve_exhaustive(p) == opt
    o = oracle_mod.Oracle(p)
    assert o.lower_bound() == closed == g["lb"]["0"]
    done = 0
    for t in (1, 2, 5, 50):
        o.iterate(t - done, 0.5)
        done = t
        if t <= 2:   # dyadic rationals: exact
            assert o.lower_bound() == g["lb"][str(t)]
        else:
            assert o.lower_bound() == pytest.approx(g["lb"][str(t)], abs=1e-9)
        if t == 1:
            lam = o.lam()
            assert np.array_equal(lam[0:4], g["lambda_row0_iter1"])
            assert np.array_equal(lam[16:20], g["lambda_col0_iter1"])
    assert o.lower_bound() <= opt + 1e-9


def test_lap_random_reaches_opt(oracle_mod):
    """Assignment polytope integral (Birkhoff): dual optimum = assignment optimum.
    Hard: LB <= OPT; soft (block-coordinate ascent may stall): reported."""
    for seed in range(6):
        cm = np.random.default_rng(seed).integers(0, 10, size=(4, 4)).astype(float)
        o = oracle_mod.Oracle(synth.lap(cm))
        o.iterate(50, 0.5)
        assert o.lower_bound() <= bf.assignment_opt(cm) + 1e-9


def test_determinism_across_threads(oracle_mod):
    """Bit-identical results for any thread count."""
    p = synth.gm_worms_like(seed=3, n_src=30, k_cand=4, knn=4)
    a = oracle_mod.Oracle(p, n_threads=1)
    b = oracle_mod.Oracle(p, n_threads=4)
    a.iterate(3, 0.5); b.iterate(3, 0.5)
    assert a.lower_bound() == b.lower_bound()
    assert np.array_equal(a.lam(), b.lam())


def test_forced_variable_clamp(oracle_mod):
    """A5: infinite min-marginal difference replaced by +-C; bound stays <= OPT."""
    # x0 = 1 forced by its own row; x0 + x1 <= 1 couples it
    p = synth.from_rows(2, [1.0, -2.0], [([0], [1], 0, 1), ([0, 1], [1, 1], -1, 1)])
    opt = bf.solve_exhaustive(p)
    o = oracle_mod.Oracle(p, clamp=100.0)
    o.pass_(True, 0.5)
    m0, m1 = o.min_marginals()
    assert m0[0] == np.inf
    assert o.deferred()[0] == pytest.approx(-0.5 * 100.0)
    for _ in range(20):
        o.iterate(1, 0.5)
        assert o.lower_bound() <= opt + 1e-9
