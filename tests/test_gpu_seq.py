"""GPU parity of the non-deferred (sequential) variant, fdog_pass_seq
(SURVEY f4), against the oracle's oracle_pass_seq, fp64, pass by
pass: lambda, the recorded min-marginals and the bound (tolerance
|a - b| <= 1e-9 (|b| + s), s = max(1, max|c|))."""
import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth

pytestmark = pytest.mark.gpu


def _s(p):
    return max(1.0, float(np.max(np.abs(p.cost))))


def _close(a, b, tol):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    ia, ib = np.isinf(a), np.isinf(b)
    assert np.array_equal(ia, ib)
    return float(np.max(np.abs(a[~ia] - b[~ib]) - tol * np.abs(b[~ib]), initial=-1.0))


def _compare(p, oracle_mod, steps, precision=64, rtol=1e-9):
    s = _s(p)
    o = oracle_mod.Oracle(p)
    g = F.Solver(p, precision=precision, record_mm=True)
    for kind, fwd, om in steps:
        if kind == "seq":
            o.pass_seq(fwd, om)
            g.pass_seq(fwd, om)
        elif kind == "def":
            o.pass_(fwd, om)
            g.pass_(fwd, om)
        else:
            o.finalize()
            g.finalize()
        assert np.max(np.abs(g.lam() - o.lam()) - rtol * np.abs(o.lam()), initial=-1) <= rtol * s, (kind, fwd)
        assert abs(g.lower_bound() - o.lower_bound()) <= rtol * (abs(o.lower_bound()) + s), (kind, fwd)
        if kind == "seq":
            assert np.all(g.deferred() == 0.0)
            gm, om_ = g.min_marginals(), o.min_marginals()
            assert _close(gm[0], om_[0], rtol) <= rtol * s and _close(gm[1], om_[1], rtol) <= rtol * s
    return g, o


SEQ6 = [("seq", t % 2 == 0, 0.5) for t in range(6)]


@pytest.mark.parametrize("name,make", [
    ("figure", synth.figure_bdd_problem),
    ("spec", synth.spec_two_constraint),
    ("lap", lambda: synth.lap(synth.LAP4_LITERAL)),
    ("gm", lambda: synth.gm_worms_like(41, n_src=50, k_cand=5, knn=6)),
    ("mrf", lambda: synth.mrf_potts(41, H=7, W=8, L=4)),
    ("qap", lambda: synth.qap(41, n=6)),
    ("ct", lambda: synth.celltrack(41, frames=4, dets=30)),
])
def test_seq_matches_oracle(oracle_mod, name, make):
    _compare(make(), oracle_mod, SEQ6)


def test_seq_random_wide_rows(oracle_mod):
    """Partitions wider than 2 (generic topology loops), ragged tiles, forced variables."""
    for seed in range(40):
        p = synth.random_ilp(700 + seed, n=10, m=7, kmax=7, coef=3, forced_ok=seed % 3 == 0)
        _compare(p, oracle_mod, SEQ6[:4])


@pytest.mark.parametrize("mode", ["rc", "tma", "stream", "rc-wide", "tma-wide"])
def test_seq_composes_with_deferred_passes(oracle_mod, monkeypatch, mode):
    """seq -> deferred -> finalize -> seq, under each sweep design (the store-design
    distances are rebuilt on the device whenever the deferred design left none);
    '-wide': tiles of 64 rows (two per lane)."""
    monkeypatch.setenv("FDOG_SWEEP", mode.split("-")[0])
    if mode.endswith("wide"):
        monkeypatch.setenv("FDOG_WIDE", "1")
        monkeypatch.setenv("FDOG_FUSED", "0")
    p = synth.gm_worms_like(43, n_src=150, k_cand=8, knn=10)
    if mode.endswith("wide"):
        assert F.Plan(p).tiles()[:, 2].max() == 64
    steps = [("seq", True, 0.5), ("seq", False, 0.5), ("def", True, 0.5), ("def", False, 0.3),
             ("fin", None, None), ("seq", False, 0.4), ("seq", True, 0.5), ("seq", False, 0.5)]
    _compare(p, oracle_mod, steps)


def test_seq_state_errors():
    p = synth.spec_two_constraint()
    g = F.Solver(p, precision=64)
    g.pass_(True, 0.5)
    with pytest.raises(F.FastdogError) as e:
        g.pass_seq(True, 0.5)       # pending deferred correction
    assert e.value.code == 6
    g.finalize()
    g.pass_seq(True, 0.5)
    with pytest.raises(F.FastdogError) as e:
        g.pass_seq(True, 1.5)
    assert e.value.code == 1


def test_seq_state_errors_after_iterate(monkeypatch):
    """The pending-correction guard also holds after fdog_iterate's fused
    single-CTA launch and after a graph-replayed iterate that follows a finalize
    (the replay path must mark delta_bar as pending too)."""
    p = synth.lap(synth.LAP4_LITERAL)  # narrow (partitions <= 2 nodes): fused-eligible
    monkeypatch.setenv("FDOG_FUSED", "1")
    g = F.Solver(p, precision=64)
    assert g.stats()["fused_small"] >= 1
    g.iterate(2, 0.5)
    with pytest.raises(F.FastdogError) as e:
        g.pass_seq(True, 0.5)
    assert e.value.code == 6
    g.finalize()
    g.pass_seq(True, 0.5)
    monkeypatch.setenv("FDOG_FUSED", "0")
    monkeypatch.setenv("FDOG_SWEEP", "tma")
    h = F.Solver(p, precision=64)
    assert h.stats()["fused_small"] == 0
    h.iterate(2, 0.5)            # captures the graph
    h.finalize()
    h.iterate(2, 0.5)            # replays it
    with pytest.raises(F.FastdogError) as e:
        h.pass_seq(True, 0.5)
    assert e.value.code == 6


def test_seq_fp32_bound(oracle_mod):
    """fp32 build: the bound after 20 sequential iterations within 1e-4 relative."""
    p = synth.gm_worms_like(45, n_src=80, k_cand=6, knn=8)
    o = oracle_mod.Oracle(p)
    g = F.Solver(p, precision=32)
    o.iterate_seq(20, 0.5)
    g.iterate_seq(20, 0.5)
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-4 * abs(o.lower_bound())


def test_seq_graph_replay_matches_direct(monkeypatch):
    """fdog_iterate_seq replays a CUDA graph of one iteration after the first:
    bit-identical to launching every level kernel directly, also after a
    deferred pass + finalize flipped the delta buffers in between."""
    p = synth.gm_worms_like(47, n_src=60, k_cand=5, knn=6)
    monkeypatch.setenv("FDOG_GRAPHS", "1")
    g1 = F.Solver(p, precision=32)
    monkeypatch.setenv("FDOG_GRAPHS", "0")
    g2 = F.Solver(p, precision=32)
    for g in (g1, g2):
        g.iterate_seq(4, 0.5)
        g.pass_(True, 0.5)
        g.finalize()
        g.iterate_seq(3, 0.5)
    assert np.array_equal(g1.lam(), g2.lam()) and g1.lower_bound() == g2.lower_bound()
    assert np.all(g1.deferred() == 0.0)
