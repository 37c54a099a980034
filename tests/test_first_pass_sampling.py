"""The sampling argument of tests/test_gpu_fullsize.py (-m "not gpu"): the
first pass from the initial state (delta_bar = 0, avg = 0) updates every
BDD independently, so on a sub-problem of sampled rows with costs
rescaled to the same initial multipliers the oracle reproduces the
full problem's lambda and delta of those rows -- here checked bit for bit
against the oracle on the whole (small) problem."""
import numpy as np
import pytest

import synth
from tests.test_gpu_fullsize import sub_problem


@pytest.mark.parametrize("make", [lambda: synth.mrf_potts(3, H=9, W=11, L=4),
                                  lambda: synth.gm_worms_like(3, n_src=40, k_cand=5, knn=5),
                                  lambda: synth.celltrack(3, frames=4, dets=25)])
@pytest.mark.parametrize("forward", [True, False])
def test_first_pass_rows_independent(oracle_mod, make, forward):
    p = make()
    o = oracle_mod.Oracle(p)
    o.pass_(forward, 0.5)
    lam, dl = o.lam(), o.deferred()
    rows = np.unique(np.random.default_rng(1).choice(p.n_cons, size=min(12, p.n_cons), replace=False))
    sub, rr = sub_problem(p, rows)
    q = oracle_mod.Oracle(sub)
    q.pass_(forward, 0.5)
    base = 0
    for j, (v, c, rel, rhs) in zip(rows, rr):
        a0, k = int(p.row_ptr[j]), len(v)
        assert np.array_equal(lam[a0:a0 + k], q.lam()[base:base + k]), j
        assert np.array_equal(dl[a0:a0 + k], q.deferred()[base:base + k]), j
        base += k
    # not true after the second pass: the averages couple the rows
    o.pass_(not forward, 0.5)
    q.pass_(not forward, 0.5)
    a0 = int(p.row_ptr[rows[0]])
    assert not all(np.array_equal(o.lam()[int(p.row_ptr[j]):int(p.row_ptr[j]) + len(r[0])],
                                  q.lam()[b:b + len(r[0])])
                   for j, r, b in zip(rows, rr, np.cumsum([0] + [len(r[0]) for r in rr])[:-1]))
