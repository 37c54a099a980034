"""Sharded solve on one GPU: W rank-solvers in one process use the
external-exchange mode of the C ABI; the test sums their exchange vectors (what
ncclAllReduce does between GPUs) and checks lambda, the bound and the deferred
min-marginals against the unsharded fp64 oracle after every pass."""
import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name,make", [
    ("gm", lambda: synth.gm_worms_like(12, n_src=60, k_cand=6, knn=6)),
    ("mrf", lambda: synth.mrf_potts(12, H=10, W=12, L=4)),
    ("qap", lambda: synth.qap(12, n=6)),
])
def test_sharded_solvers_match_unsharded(oracle_mod, world, name, make):
    p = make()
    s = max(1.0, float(np.abs(p.cost).max()))
    ranks = [F.Solver(p, precision=64, rank=r, world=world) for r in range(world)]
    assert sum(g.num_slots() for g in ranks) == int(p.row_ptr[-1])
    o = oracle_mod.Oracle(p)
    assert abs(sum(g.lower_bound() for g in ranks) - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    for t in range(6):
        fwd = t % 2 == 0
        for g in ranks:
            g.pass_begin(fwd, 0.5)
        x = sum(g.exchange_read() for g in ranks)
        for g in ranks:
            g.exchange_write(x)
        for g in ranks:
            g.pass_end(fwd, 0.5)
        o.pass_(fwd, 0.5)
        lam = np.full(o.num_slots(), np.nan)
        dl = np.full(o.num_slots(), np.nan)
        for g in ranks:
            con, pos = g.slot_index()
            idx = p.row_ptr[con] + pos
            lam[idx] = g.lam()
            dl[idx] = g.deferred()
        assert not np.isnan(lam).any()
        assert np.max(np.abs(lam - o.lam())) <= 1e-9 * s, f"pass {t}"
        assert np.max(np.abs(dl - o.deferred())) <= 1e-9 * s
        lb = sum(g.lower_bound() for g in ranks)
        assert abs(lb - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    with pytest.raises(F.FastdogError) as e:
        ranks[0].iterate(1, 0.5)
    assert e.value.code == 6
