"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star):
  * fp64 build after 1 iteration: |a - b| <= 1e-9 * (|b| + s), s = max(1, max|c|),
    on lambda, (m0, m1), delta_bar and the lower bound;
  * fp32 build after 100 iterations: lower bound within 1e-4 relative;
  * dyadic instances (LAP literal, iterations 1-2): bit-exact in fp64 and fp32;
  * node / arc counts: exact (tests/test_host.py and below).
"""
import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth

pytestmark = pytest.mark.gpu


def _s(problem):
    return max(1.0, float(np.max(np.abs(problem.cost))) if problem.n_vars else 1.0)


def _close(a, b, tol):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    inf_a, inf_b = np.isinf(a), np.isinf(b)
    assert np.array_equal(inf_a, inf_b), "infinite min-marginals differ"
    assert np.array_equal(np.sign(a[inf_a]), np.sign(b[inf_b]))
    fa, fb = a[~inf_a], b[~inf_b]
    err = np.abs(fa - fb) - tol * np.abs(fb)
    return float(err.max()) if err.size else -1.0


def _compare_pass_by_pass(problem, oracle_mod, passes, precision=64, rtol=1e-9, omega=0.5):
    s = _s(problem)
    o = oracle_mod.Oracle(problem)
    g = F.Solver(problem, precision=precision, record_mm=True)
    assert g.num_slots() == o.num_slots()
    con, pos = g.slot_index()
    assert np.array_equal(con, np.repeat(np.arange(problem.n_cons), np.diff(problem.row_ptr)))
    abs_tol = rtol * s
    assert abs(g.lower_bound() - o.lower_bound()) <= rtol * (abs(o.lower_bound()) + s)
    for t in range(passes):
        fwd = t % 2 == 0
        o.pass_(fwd, omega)
        g.pass_(fwd, omega)
        for name, a, b in (("lambda", g.lam(), o.lam()), ("delta", g.deferred(), o.deferred())):
            err = np.abs(a - b) - rtol * np.abs(b)
            assert err.max(initial=-1) <= abs_tol, f"pass {t} {name}: max err {np.max(np.abs(a - b))}"
        gm0, gm1 = g.min_marginals()
        om0, om1 = o.min_marginals()
        assert _close(gm0, om0, rtol) <= abs_tol, f"pass {t} m0"
        assert _close(gm1, om1, rtol) <= abs_tol, f"pass {t} m1"
        lb_g, lb_o = g.lower_bound(), o.lower_bound()
        assert abs(lb_g - lb_o) <= rtol * (abs(lb_o) + s), f"pass {t} lb {lb_g} vs {lb_o}"
    return g, o


def test_figure_example(oracle_mod):
    _compare_pass_by_pass(synth.figure_bdd_problem(), oracle_mod, passes=4)


def test_spec_two_constraint(oracle_mod):
    _compare_pass_by_pass(synth.spec_two_constraint(), oracle_mod, passes=20)


@pytest.mark.parametrize("precision", [64, 32])
def test_lap4_literal_bit_exact(oracle_mod, precision):
    """Iterations 1-2 on the literal LAP are dyadic rationals: bit-exact."""
    p = synth.lap(synth.LAP4_LITERAL)
    o = oracle_mod.Oracle(p)
    g = F.Solver(p, precision=precision, record_mm=True)
    assert g.lower_bound() == o.lower_bound() == 6.5
    for t in range(4):
        o.pass_(t % 2 == 0, 0.5)
        g.pass_(t % 2 == 0, 0.5)
        assert np.array_equal(g.lam(), o.lam())
        assert np.array_equal(g.deferred(), o.deferred())
        assert g.lower_bound() == o.lower_bound()
    assert g.lower_bound() == 8.109375
    if precision == 64:
        g.iterate(48, 0.5)
        assert g.lower_bound() == pytest.approx(10.0, abs=1e-9)


def test_random_tiny_ilps_fp64(oracle_mod):
    """200 random tiny ILPs (ragged tiles, per-lane topologies), 1 iteration, fp64."""
    for seed in range(200):
        p = synth.random_ilp(seed, n=10, m=7, kmax=7, coef=3)
        _compare_pass_by_pass(p, oracle_mod, passes=2)


def test_random_ilps_with_forced_vars(oracle_mod):
    """Forced variables: infinite min-marginals and the clamp (A5), fp64."""
    for seed in range(30):
        p = synth.random_ilp(900 + seed, n=8, m=6, kmax=5, coef=3, forced_ok=True)
        _compare_pass_by_pass(p, oracle_mod, passes=4)


@pytest.mark.parametrize("name,make", [
    ("gm", lambda: synth.gm_worms_like(4, n_src=80, k_cand=6, knn=8)),
    ("mrf", lambda: synth.mrf_potts(4, H=12, W=14, L=4)),
    ("mrf_cut", lambda: synth.mrf_potts_cut(4, H=12, W=14, L=4)),
    ("qap", lambda: synth.qap(4, n=7)),
    ("celltrack", lambda: synth.celltrack(4, frames=5, dets=40)),
    ("wide_rows", lambda: synth.random_ilp(7, n=40, m=60, kmax=12, coef=5)),
    ("gap", lambda: synth.gap(4, jobs=40, agents=5)),
    ("mckp", lambda: synth.mckp(4, classes=200, knaps=12, k=20)),
])
def test_workload_shapes_fp64(oracle_mod, name, make):
    """Several tiles, ragged tails, both tile kinds: 1 iteration element-wise, then 10 more."""
    p = make()
    g, o = _compare_pass_by_pass(p, oracle_mod, passes=2)
    g.iterate(10, 0.5)
    o.iterate(10, 0.5)
    s = _s(p)
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-8 * (abs(o.lower_bound()) + s)
    assert np.allclose(g.lam(), o.lam(), rtol=1e-8, atol=1e-8 * s)


@pytest.mark.parametrize("name,make", [
    ("lap4", lambda: synth.lap_random(4, 0)),
    ("gm", lambda: synth.gm_worms_like(5, n_src=120, k_cand=8, knn=10)),
    ("mrf", lambda: synth.mrf_potts(5, H=20, W=20, L=5)),
    ("mrf_cut", lambda: synth.mrf_potts_cut(5, H=20, W=20, L=5)),
    ("qap", lambda: synth.qap(5, n=8)),
    ("gap", lambda: synth.gap(5, jobs=40, agents=5)),
    ("mckp", lambda: synth.mckp(5, classes=200, knaps=12, k=20)),
])
def test_fp32_lower_bound_100_iterations(oracle_mod, name, make):
    """fp32 build: LB within 1e-4 relative after 100 iterations; monotone within
    1e-6 (1 + |LB|) (Prop. 1)."""
    p = make()
    o = oracle_mod.Oracle(p)
    g = F.Solver(p, precision=32)
    lbs = [g.lower_bound()]
    for _ in range(10):
        g.iterate(10, 0.5)
        lbs.append(g.lower_bound())
    o.iterate(100, 0.5)
    lb_o = o.lower_bound()
    assert abs(lbs[-1] - lb_o) <= 1e-4 * max(abs(lb_o), 1.0), f"{lbs[-1]} vs {lb_o}"
    lbs = np.array(lbs)
    assert np.all(np.diff(lbs) >= -1e-6 * (1 + np.abs(lbs[:-1])))


def test_finalize_feasible(oracle_mod):
    """after finalize sum_j lambda_i^j = c_i, bound = sum_j E^j (I5)."""
    p = synth.gm_worms_like(6, n_src=50, k_cand=5, knn=6)
    g = F.Solver(p, precision=64)
    o = oracle_mod.Oracle(p)
    g.iterate(7, 0.5); o.iterate(7, 0.5)
    g.finalize(); o.finalize()
    lam = g.lam()
    acc = np.zeros(p.n_vars)
    np.add.at(acc, p.col_var, lam)
    used = np.bincount(p.col_var, minlength=p.n_vars) > 0
    assert np.max(np.abs(acc - p.cost)[used]) < 1e-9 * _s(p)
    assert g.lower_bound() == pytest.approx(o.lower_bound(), rel=1e-9, abs=1e-9)
    # iterate again after finalize (restart from feasible lambda with mbar = 0)
    g.iterate(2, 0.5); o.iterate(2, 0.5)
    assert g.lower_bound() == pytest.approx(o.lower_bound(), rel=1e-9, abs=1e-9)


def test_finalize_averaged(oracle_mod):
    """Averaged final correction (P:673 prose) vs the oracle; feasible afterwards."""
    p = synth.gm_worms_like(15, n_src=50, k_cand=5, knn=6)
    g = F.Solver(p, precision=64)
    o = oracle_mod.Oracle(p)
    g.iterate(5, 0.5); o.iterate(5, 0.5)
    g.pass_(True, 0.5); o.pass_(True, 0.5)
    g.finalize(averaged=True); o.finalize(averaged=True)
    s = _s(p)
    assert np.max(np.abs(g.lam() - o.lam())) <= 1e-9 * s
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    assert np.all(g.deferred() == 0)
    g.iterate(2, 0.5); o.iterate(2, 0.5)
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)


def test_edge_cases(oracle_mod):
    # no constraints: bound = sum min(c, 0)
    p = synth.from_rows(3, [-1.0, 2.0, -0.5], [])
    g = F.Solver(p, precision=64)
    assert g.lower_bound() == -1.5 and g.num_slots() == 0
    g.iterate(2, 0.5)
    assert g.lower_bound() == -1.5
    # single one-variable row + a free variable
    p = synth.from_rows(2, [3.0, -1.0], [([0], [1], 1, 1)])
    _compare_pass_by_pass(p, oracle_mod, passes=4)
    # 33 identical rows: one shared-topology tile + one ragged per-lane tile
    rows = [([i, i + 1, i + 2], [1, 1, 1], 0, 1) for i in range(33)]
    p = synth.from_rows(35, np.linspace(-1, 1, 35), rows)
    g, _ = _compare_pass_by_pass(p, oracle_mod, passes=4)
    st = g.stats()
    assert st["tiles"] == 2 and st["tiles_shared_topology"] == 1
    # omega = 1 and omega small
    _compare_pass_by_pass(synth.spec_two_constraint(), oracle_mod, passes=4, omega=1.0)
    _compare_pass_by_pass(synth.spec_two_constraint(), oracle_mod, passes=4, omega=0.1)


def test_unusual_pass_orders(oracle_mod):
    """Backward first, two forwards in a row, pass after finalize: the distances
    of the opposite direction are recomputed when needed."""
    p = synth.gm_worms_like(8, n_src=40, k_cand=5, knn=6)
    s = _s(p)
    o = oracle_mod.Oracle(p)
    g = F.Solver(p, precision=64)
    for fwd in (False, True, True, False, False, True):
        o.pass_(fwd, 0.5)
        g.pass_(fwd, 0.5)
        assert np.max(np.abs(g.lam() - o.lam())) <= 1e-9 * s
        assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    o.finalize(); g.finalize()
    o.pass_(False, 0.5); g.pass_(False, 0.5)
    assert np.max(np.abs(g.lam() - o.lam())) <= 1e-9 * s


def test_graph_replay_matches_direct_launches(monkeypatch):
    """fdog_iterate's CUDA-graph replay gives bit-identical results to launching
    the kernels one by one (same kernels, same order, deterministic reductions)."""
    p = synth.gm_worms_like(9, n_src=60, k_cand=6, knn=6)
    monkeypatch.setenv("FDOG_FUSED", "0")
    monkeypatch.setenv("FDOG_GRAPHS", "1")
    g1 = F.Solver(p, precision=32)
    monkeypatch.setenv("FDOG_GRAPHS", "0")
    g2 = F.Solver(p, precision=32)
    for n, om in ((3, 0.5), (2, 0.3), (1, 0.5), (1, 0.5)):
        g1.iterate(n, om); g2.iterate(n, om)
        assert np.array_equal(g1.lam(), g2.lam()) and g1.lower_bound() == g2.lower_bound()
    g1.pass_(True, 0.5); g2.pass_(True, 0.5)      # odd parity, then graphs again
    g1.iterate(2, 0.5); g2.iterate(2, 0.5)
    assert np.array_equal(g1.lam(), g2.lam()) and np.array_equal(g1.deferred(), g2.deferred())
    g1.profile_enable(True)                        # events on: direct launches
    g1.iterate(1, 0.5); g2.iterate(1, 0.5)
    assert np.array_equal(g1.lam(), g2.lam())
    assert "sweep_forward" in g1.profile()


@pytest.mark.parametrize("resident", ["0", "1"])
@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("name,make", [
    ("lap", lambda: synth.lap(synth.LAP4_LITERAL)),
    ("lap_random", lambda: synth.lap_random(9, 5)),
    ("gm", lambda: synth.gm_worms_like(21, n_src=50, k_cand=5, knn=6)),
    ("mrf", lambda: synth.mrf_potts(21, H=7, W=9, L=3)),
    ("ct", lambda: synth.celltrack(21, frames=3, dets=30)),
])
def test_fused_small_path(oracle_mod, monkeypatch, resident, precision, name, make):
    """Small narrow problems run every iteration of fdog_iterate in one
    single-CTA launch (fused_small_kernel; state in global memory, or copied
    into shared memory when it fits).  Same arithmetic as the per-pass
    kernels: bit-identical lambda, delta_bar, min-marginals and bound, and the
    oracle's iterates within the fp64 tolerance."""
    p = make()
    monkeypatch.setenv("FDOG_FUSED_SMEM", resident)
    monkeypatch.setenv("FDOG_FUSED", "1")
    gf = F.Solver(p, precision=precision, record_mm=True)
    monkeypatch.setenv("FDOG_FUSED", "0")
    monkeypatch.setenv("FDOG_SWEEP", "tma")  # same (store-design) tile packing as the fused path
    gd = F.Solver(p, precision=precision, record_mm=True)
    assert gf.stats()["fused_small"] >= 1 and gd.stats()["fused_small"] == 0
    if resident == "0":
        assert gf.stats()["fused_small"] == 1
    o = oracle_mod.Oracle(p)
    s = _s(p)
    for n, om in ((1, 0.5), (3, 0.3), (2, 0.5)):
        l0 = gf.stats()["launches"]
        gf.iterate(n, om); gd.iterate(n, om); o.iterate(n, om)
        assert gf.stats()["launches"] == l0 + 1
        assert np.array_equal(gf.lam(), gd.lam()) and np.array_equal(gf.deferred(), gd.deferred())
        m_f, m_d = gf.min_marginals(), gd.min_marginals()
        assert np.array_equal(m_f[0], m_d[0]) and np.array_equal(m_f[1], m_d[1])
        assert gf.lower_bound() == gd.lower_bound()
        if precision == 64:
            # the north_star fp64 tolerance, |a - b| <= 1e-9 (|b| + s),
            # on lambda, delta_bar, the min-marginals and the bound after every call
            b = o.lam()
            assert np.all(np.abs(gf.lam() - b) <= 1e-9 * (np.abs(b) + s))
            b = o.deferred()
            assert np.all(np.abs(gf.deferred() - b) <= 1e-9 * (np.abs(b) + s))
            for x, y in zip(m_f, o.min_marginals()):
                fin = np.isfinite(y)
                assert np.array_equal(np.isfinite(x), fin)
                assert np.all(np.abs(x[fin] - y[fin]) <= 1e-9 * (np.abs(y[fin]) + s))
            assert abs(gf.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    gf.pass_(True, 0.5); gd.pass_(True, 0.5)      # odd parity, then fused again
    gf.iterate(2, 0.5); gd.iterate(2, 0.5)
    assert np.array_equal(gf.lam(), gd.lam()) and gf.lower_bound() == gd.lower_bound()


_SWEEP_CASES = [
    ("gm", lambda: synth.gm_worms_like(13, n_src=70, k_cand=6, knn=8)),
    ("mrf", lambda: synth.mrf_potts(13, H=9, W=11, L=4)),
    ("qap", lambda: synth.qap(13, n=8)),
    ("ct", lambda: synth.celltrack(13, frames=4, dets=40)),
    ("lap", lambda: synth.lap(synth.LAP4_LITERAL)),
]


@pytest.mark.parametrize("mode", ["rc", "tma", "stream"])
@pytest.mark.parametrize("name,make", _SWEEP_CASES)
def test_all_sweep_kernels(oracle_mod, monkeypatch, mode, name, make):
    """The three sweep designs -- recompute (the default for narrow problems:
    distances of the opposite direction rebuilt on chip), TMA-staged store and
    streaming store -- each match the oracle pass by pass, fp64."""
    monkeypatch.setenv("FDOG_SWEEP", mode)
    g, _ = _compare_pass_by_pass(make(), oracle_mod, passes=6)
    st = g.stats()
    assert st["sweep_streaming"] == (1 if mode == "stream" else 0)
    assert st["sweep_recompute"] == (1 if mode == "rc" else 0)


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("name,make", _SWEEP_CASES[:4])
def test_recompute_equals_store_bitwise(monkeypatch, precision, name, make):
    """The recomputed distances equal the stored ones exactly (lambda has not
    changed since the previous pass computed them, same operations in the same
    order), so the recompute and store designs give bit-identical iterates --
    including after unusual pass orders, finalize and set_state.  (The bound
    is a sum of per-tile partials in tile order: equal up to summation order.)"""
    p = make()
    gs = {}
    for mode in ("rc", "tma", "stream"):
        monkeypatch.setenv("FDOG_SWEEP", mode)
        monkeypatch.setenv("FDOG_FUSED", "0")
        gs[mode] = F.Solver(p, precision=precision, record_mm=True)
    assert gs["rc"].stats()["sweep_recompute"] == 1
    def lb_close(a, b):  # the per-tile partials are summed in tile order, and
        return abs(a - b) <= 1e-12 * (1 + abs(b))  # the two designs pack tiles differently
    lb0 = {m: g.lower_bound() for m, g in gs.items()}
    assert lb_close(lb0["rc"], lb0["tma"]) and lb_close(lb0["stream"], lb0["tma"])
    steps = [("it", 3, 0.5), ("pass", True, 0.5), ("pass", True, 0.3), ("pass", False, 0.5),
             ("pass", False, 0.5), ("it", 2, 0.4), ("fin",), ("it", 2, 0.5)]
    for st in steps:
        for g in gs.values():
            if st[0] == "it":
                g.iterate(st[1], st[2])
            elif st[0] == "pass":
                g.pass_(st[1], st[2])
            else:
                g.finalize()
        ref = gs["tma"]
        for m in ("rc", "stream"):
            g = gs[m]
            assert np.array_equal(g.lam(), ref.lam()), (m, st)
            assert np.array_equal(g.deferred(), ref.deferred()), (m, st)
            assert lb_close(g.lower_bound(), ref.lower_bound()), (m, st)
            if st[0] != "fin":
                a, b = g.min_marginals(), ref.min_marginals()
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), (m, st)
    lam, dl = gs["tma"].lam(), gs["tma"].deferred()
    for g in gs.values():
        g.set_state(lam, dl)
        g.iterate(1, 0.5)
    assert np.array_equal(gs["rc"].lam(), gs["tma"].lam())


@pytest.mark.parametrize("mode", ["rc", "tma"])
@pytest.mark.parametrize("name,make", _SWEEP_CASES[:4])
def test_stage_buffers_bitwise(oracle_mod, monkeypatch, mode, name, make):
    """Single- and double-buffered stages (FDOG_NBUF; the plan's default
    differs per design and problem) give bit-identical iterates: a BDD's
    arithmetic does not depend on the tile it is packed into.  One of them
    against the oracle (fp64)."""
    p = make()
    monkeypatch.setenv("FDOG_SWEEP", mode)
    monkeypatch.setenv("FDOG_FUSED", "0")
    gs = []
    for nb in ("1", "2"):
        monkeypatch.setenv("FDOG_NBUF", nb)
        gs.append(F.Solver(p, precision=64))
    assert gs[0].stats()["sweep_smem_per_warp"] < gs[1].stats()["sweep_smem_per_warp"]
    o = oracle_mod.Oracle(p)
    s = _s(p)
    for t in range(4):
        fwd = t % 2 == 0
        for g in gs:
            g.pass_(fwd, 0.5)
        o.pass_(fwd, 0.5)
        assert np.array_equal(gs[0].lam(), gs[1].lam()) and np.array_equal(gs[0].deferred(), gs[1].deferred())
        assert np.max(np.abs(gs[0].lam() - o.lam())) <= 1e-9 * s
        assert abs(gs[0].lower_bound() - gs[1].lower_bound()) <= 1e-12 * (1 + abs(o.lower_bound()))
    gs[0].iterate(2, 0.5)
    gs[1].iterate(2, 0.5)
    assert np.array_equal(gs[0].lam(), gs[1].lam())


def _same_bound(g0, g1):
    a, b = g0.lower_bound(), g1.lower_bound()
    return abs(a - b) <= 1e-12 * (1 + abs(b))


@pytest.mark.parametrize("mode", ["rc", "tma"])
@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("name,make", [
    ("mrf4", lambda: synth.mrf_potts(8, H=20, W=24, L=4)),
    ("mrf8", lambda: synth.mrf_potts(8, H=10, W=12, L=8)),
    ("gm8", lambda: synth.gm_worms_like(8, n_src=60, k_cand=7, knn=6)),
])
def test_tile_pairs_bitwise(oracle_mod, monkeypatch, mode, precision, name, make):
    """Tile-closed pairs (|J_i| = 2, both slots in one tile) averaged on chip by
    the sweep equal the averaging kernel's ELL path bit for bit (same
    arithmetic, (d1 + d2) / 2): FDOG_PAIRS=0 vs the default, pass by pass and
    through the graph-replayed iterate; the bound, finalize(averaged) and the
    oracle (fp64) as well.  (Instances whose bundles -- 2 L marginalisation
    rows per edge -- divide a 32-row tile, so the packer picks bundle order.)"""
    p = make()
    monkeypatch.setenv("FDOG_SWEEP", mode)
    monkeypatch.setenv("FDOG_FUSED", "0")
    monkeypatch.setenv("FDOG_PAIRS", "0")
    g0 = F.Solver(p, precision=precision)
    monkeypatch.delenv("FDOG_PAIRS")
    g1 = F.Solver(p, precision=precision)
    assert g0.stats()["tile_pairs"] == 0 and g1.stats()["tile_pairs"] > 0
    o = oracle_mod.Oracle(p)
    s = _s(p)
    for t in range(4):
        fwd = t % 2 == 0
        g0.pass_(fwd, 0.5)
        g1.pass_(fwd, 0.5)
        o.pass_(fwd, 0.5)
        assert np.array_equal(g0.lam(), g1.lam()) and np.array_equal(g0.deferred(), g1.deferred())
        assert _same_bound(g0, g1)
        if precision == 64:
            assert np.max(np.abs(g1.lam() - o.lam())) <= 1e-9 * s
    g0.iterate(3, 0.5)
    g1.iterate(3, 0.5)
    assert np.array_equal(g0.lam(), g1.lam()) and _same_bound(g0, g1)
    g0.finalize(averaged=True)
    g1.finalize(averaged=True)
    assert np.array_equal(g0.lam(), g1.lam()) and _same_bound(g0, g1)
    g0.iterate(2, 0.5)
    g1.iterate(2, 0.5)
    assert np.array_equal(g0.lam(), g1.lam())


def test_tile_schedules_bitwise(monkeypatch):
    """Static round-robin, dynamic claims of one tile and batched claims of
    several tiles per atomic give bit-identical iterates and bounds (a BDD's
    arithmetic does not depend on the warp that runs it; the bound sums the
    per-tile partials in tile order).  One warp per CTA, so every warp runs
    several tiles and the batches are exercised."""
    p = synth.mrf_potts(5, H=100, W=100, L=8)
    monkeypatch.setenv("FDOG_WPB", "1")
    gs = {}
    for name, env in (("static", {"FDOG_SCHED": "static"}), ("claim1", {"FDOG_SCHED": "dynamic", "FDOG_CLAIM": "1"}),
                      ("claim3", {"FDOG_SCHED": "dynamic", "FDOG_CLAIM": "3"})):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        gs[name] = F.Solver(p, precision=32)
        for k in env:
            monkeypatch.delenv(k)
    st = gs["claim3"].stats()
    assert st["tiles"] > 2 * st["sweep_grid"]
    for g in gs.values():
        g.iterate(3, 0.5)
        g.pass_(True, 0.5)
    ref = gs["static"]
    for g in gs.values():
        assert np.array_equal(g.lam(), ref.lam()) and np.array_equal(g.deferred(), ref.deferred())
        assert g.lower_bound() == ref.lower_bound()


def test_errors_and_state():
    p = synth.spec_two_constraint()
    g = F.Solver(p, precision=64)
    with pytest.raises(F.FastdogError) as e:
        g.min_marginals()
    assert e.value.code == 6
    with pytest.raises(F.FastdogError) as e:
        g.iterate(1, 1.5)
    assert e.value.code == 1
    g.iterate(3, 0.5)
    lam, dl, lb = g.lam(), g.deferred(), g.lower_bound()
    h = F.Solver(p, precision=64)
    h.set_state(lam, dl)            # checkpoint / resume
    assert np.array_equal(h.lam(), lam) and np.array_equal(h.deferred(), dl)
    # the resumed bound is the lifted bound (A7) with its outstanding
    # sum min(delta_bar, 0) term, not the raw sum_j E^j
    assert np.any(dl < 0)
    assert h.lower_bound() == pytest.approx(lb, rel=1e-12, abs=1e-12)
    g.iterate(2, 0.5); h.iterate(2, 0.5)
    assert np.array_equal(g.lam(), h.lam()) and g.lower_bound() == h.lower_bound()
    with pytest.raises(F.FastdogError) as e:
        F.Solver(synth.from_rows(2, [0, 0], [([0, 1], [1, 1], -1, -1)]))
    assert e.value.code == 2


def test_full_size_gm_fp32(oracle_mod):
    """BASELINE configs[1] at full size in bench.py's launch configuration (fp32):
    lambda after 1 iteration vs the oracle (fp64) element-wise at fp32 tolerance,
    bound after 100 iterations within 1e-4 relative (north_star), node/arc
    counts exact."""
    p = synth.gm_worms_like(0)
    g = F.Solver(p, precision=32)
    o = oracle_mod.Oracle(p)
    st = g.stats()
    assert st["nodes"] == o.total_nodes() and st["arcs"] == 2 * o.total_nodes()
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-6 * abs(o.lower_bound())
    g.iterate(1, 0.5); o.iterate(1, 0.5)
    s = _s(p)
    a, b = g.lam(), o.lam()
    assert np.max(np.abs(a - b) - 1e-5 * np.abs(b)) <= 1e-5 * s
    g.iterate(99, 0.5); o.iterate(99, 0.5)
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-4 * abs(o.lower_bound())


def test_full_size_gm_fp64_sampled(oracle_mod):
    """fp64 at full GM size: every slot after 1 iteration within 1e-9 (the oracle
    finishes the whole instance in seconds)."""
    p = synth.gm_worms_like(0)
    g = F.Solver(p, precision=64)
    o = oracle_mod.Oracle(p)
    g.iterate(1, 0.5); o.iterate(1, 0.5)
    s = _s(p)
    a, b = g.lam(), o.lam()
    assert np.max(np.abs(a - b) - 1e-9 * np.abs(b)) <= 1e-9 * s
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)


def test_concurrent_solvers_with_different_budgets(oracle_mod):
    """Several solvers alive in one process with different per-warp shared-memory
    budgets and sweep designs (the dynamic shared-memory limit is a
    per-function attribute shared by all of them): interleaved passes, each
    still matches its own oracle."""
    probs = [synth.gm_worms_like(31, n_src=50, k_cand=6, knn=6), synth.qap(31, n=7),
             synth.mrf_potts(31, H=8, W=9, L=5), synth.random_ilp(31, n=30, m=40, kmax=9, coef=4)]
    gs = [F.Solver(p, precision=64) for p in probs]
    os_ = [oracle_mod.Oracle(p) for p in probs]
    budgets = {g.stats()["sweep_smem_per_warp"] for g in gs}
    assert len(budgets) > 1
    for t in range(4):
        for g, o in zip(gs, os_):
            g.pass_(t % 2 == 0, 0.5)
            o.pass_(t % 2 == 0, 0.5)
    for g, o, p in zip(gs, os_, probs):
        s = _s(p)
        assert np.max(np.abs(g.lam() - o.lam())) <= 1e-9 * s
        assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)


def _long_rows(seed, n=2560, rows=7):
    """Rows too long to stage whole: one-hot / at-most-one rows over 900-2400
    of n variables (several rows share a shape, so tiles hold several lanes),
    plus short rows, so every variable is shared."""
    rng = np.random.default_rng(seed)
    out = []
    for r in range(rows):
        k = [900, 900, 2400, 1500, 900, 2400, 1500][r % 7]
        v = np.sort(rng.choice(n, size=k, replace=False))
        out.append((v, np.ones(k), synth.EQ if r % 2 else synth.LE, 1))
    for q in range(0, n - 1, 2):
        out.append((np.array([q, q + 1]), np.ones(2), synth.LE, 1))
    return synth.from_rows(n, rng.uniform(-1, 1, size=n).round(3), out, f"long_rows({seed})")


@pytest.mark.parametrize("chunk", ["1", "0"])
def test_long_rows_chunked(oracle_mod, monkeypatch, chunk):
    """Rows too long to stage whole run the chunked kernel (partitions walked
    through shared memory in chunks, state carried across chunks) -- or the
    streaming kernel with FDOG_CHUNK=0; both match the oracle pass by pass, fp64.
    Includes the thin-hop microbench's single 3000-partition row."""
    monkeypatch.setenv("FDOG_CHUNK", chunk)
    for p in (_long_rows(3), synth.thin_hop(5, k=3000)):
        g, _ = _compare_pass_by_pass(p, oracle_mod, passes=4)
        assert g.stats()["sweep_streaming"] == (2 if chunk == "1" else 1)


def test_nccl_one_rank_communicator(monkeypatch):
    """The NCCL path of a multi-GPU run (dlopen of the torch-bundled libnccl,
    ncclCommInitRank with a torch-generated unique id, ncclAllReduce on the
    solver's stream, ncclCommDestroy) on a one-rank communicator: the bound's
    allreduce over one rank is the identity."""
    import os
    import torch
    import nvidia.nccl
    lib = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
    p = synth.gm_worms_like(51, n_src=40, k_cand=5, knn=6)
    monkeypatch.setenv("FDOG_NCCL_SELF", "1")
    g = F.Solver(p, precision=64, nccl_unique_id=torch.cuda.nccl.unique_id(), nccl_library=lib)
    monkeypatch.setenv("FDOG_NCCL_SELF", "0")
    h = F.Solver(p, precision=64)
    for _ in range(3):
        g.iterate(1, 0.5); h.iterate(1, 0.5)
        assert g.lower_bound() == h.lower_bound()
    g.close()


def _max_lanes(p, precision, monkeypatch=None):
    return int(F.Plan(p, precision=precision).tiles()[:, 2].max())


@pytest.mark.parametrize("mode", ["rc", "tma"])
@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("name,make,lanes", [
    ("mrf", lambda: synth.mrf_potts(9, H=20, W=24, L=4), 128),         # K = 4 rows: 4 per lane (fp32)
    ("mrf8", lambda: synth.mrf_potts(9, H=12, W=12, L=8), 64),         # K = 8 / 9 rows: 2 per lane
    ("mrf_cut", lambda: synth.mrf_potts_cut(9, H=16, W=18, L=5), 128),  # K = 3 rows: 4 per lane (fp32)
    ("gm", lambda: synth.gm_worms_like(9, n_src=150, k_cand=8, knn=10), 64),
])
def test_wide_tiles_bitwise(oracle_mod, monkeypatch, mode, precision, name, make, lanes):
    """Tiles of 32 R rows (R rows per lane, kernels.cu mask_tile) run each row's
    arithmetic exactly as 32-row tiles: FDOG_WIDE=0 vs the default, pass by pass
    (lambda, delta_bar, min-marginals bit for bit; the bound at 1e-12, its
    per-tile partials are summed in another order), through the graph-replayed
    iterate, finalize and a restart; fp64 against the oracle at 1e-9."""
    p = make()
    monkeypatch.setenv("FDOG_SWEEP", mode)
    monkeypatch.setenv("FDOG_FUSED", "0")
    monkeypatch.setenv("FDOG_WIDE", "1")  # whenever eligible (the default asks the budget model)
    want = lanes if precision == 32 else min(lanes, 64)
    assert _max_lanes(p, precision) == want
    g1 = F.Solver(p, precision=precision, record_mm=True)
    monkeypatch.setenv("FDOG_WIDE", "0")
    assert _max_lanes(p, precision) == 32
    g0 = F.Solver(p, precision=precision, record_mm=True)
    o = oracle_mod.Oracle(p)
    s = _s(p)
    for t in range(4):
        fwd = t % 2 == 0
        for g in (g0, g1, o):
            g.pass_(fwd, 0.5)
        assert np.array_equal(g0.lam(), g1.lam()) and np.array_equal(g0.deferred(), g1.deferred())
        for a, b in zip(g0.min_marginals(), g1.min_marginals()):
            assert np.array_equal(a, b)
        assert _same_bound(g0, g1)
        if precision == 64:
            assert np.max(np.abs(g1.lam() - o.lam())) <= 1e-9 * s
            assert abs(g1.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    for g in (g0, g1):
        g.iterate(3, 0.5)
    assert np.array_equal(g0.lam(), g1.lam()) and _same_bound(g0, g1)
    for g in (g0, g1):
        g.finalize()
        g.iterate(2, 0.5)
    assert np.array_equal(g0.lam(), g1.lam()) and _same_bound(g0, g1)


def test_cooperative_wide_bdds(oracle_mod):
    """Knapsack rows wider than 32 nodes per partition run node-parallel (one
    warp per BDD, warp-shuffle min-marginals, atomic-min relaxation):
    a generalized assignment instance with 130 k-node capacity BDDs (beyond the
    16-bit codes of lane tiles), fp64, every slot, min-marginals and the bound
    after every pass for two iterations at 1e-9; then 10 more iterations; the
    non-deferred variant refuses such BDDs."""
    p = synth.gap(6, jobs=300, agents=20)
    g, o = _compare_pass_by_pass(p, oracle_mod, passes=4)
    t = F.Plan(p).tiles()
    assert ((t[:, 0] & 32) != 0).sum() == 20 and t[:, 4].max() > 65534
    g.iterate(10, 0.5)
    o.iterate(10, 0.5)
    s = _s(p)
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-8 * (abs(o.lower_bound()) + s)
    assert np.allclose(g.lam(), o.lam(), rtol=1e-8, atol=1e-8 * s)
    with pytest.raises(F.FastdogError) as e:
        g.pass_seq(True, 0.5)
    assert e.value.code == 1


def test_cooperative_unusual_orders_and_finalize(oracle_mod):
    """Cooperative tiles through the distance recomputes (backward first, two
    forwards: kEnergy / kCfr sweeps), finalize and the averaged finalize."""
    p = synth.mckp(7, classes=300, knaps=20, k=24)
    o = oracle_mod.Oracle(p)
    g = F.Solver(p, precision=64, record_mm=True)
    s = _s(p)
    for fwd in (False, False, True, True, False):
        g.pass_(fwd, 0.5)
        o.pass_(fwd, 0.5)
        assert np.max(np.abs(g.lam() - o.lam())) <= 1e-9 * s
        assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    g.finalize()
    o.finalize()
    assert np.max(np.abs(g.lam() - o.lam())) <= 1e-9 * s
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    g.iterate(3, 0.5)
    o.iterate(3, 0.5)
    g.finalize(averaged=True)
    o.finalize(averaged=True)
    assert np.max(np.abs(g.lam() - o.lam())) <= 1e-9 * s


@pytest.mark.parametrize("name,make", [
    ("qap", lambda: synth.qap(16, n=12)),
    ("celltrack", lambda: synth.celltrack(16, frames=8, dets=60)),
    ("gm", lambda: synth.gm_worms_like(16, n_src=120, k_cand=8, knn=10)),
])
def test_tmem_distances_bitwise(monkeypatch, name, make):
    """Recompute design, fp32: the distance scratch of 32-row tiles in tensor
    memory (tcgen05.st / tcgen05.ld, kernels.cu TmemD) equals the shared-memory
    scratch bit for bit (FDOG_TMEM=1 vs 0) -- lambda, delta_bar and the
    min-marginals pass by pass, then through the graph-replayed iterate."""
    p = make()
    monkeypatch.setenv("FDOG_SWEEP", "rc")
    monkeypatch.setenv("FDOG_FUSED", "0")
    monkeypatch.setenv("FDOG_TMEM", "1")
    g1 = F.Solver(p, precision=32, record_mm=True)
    assert g1.stats()["tmem_cols"] >= 32
    monkeypatch.setenv("FDOG_TMEM", "0")
    g0 = F.Solver(p, precision=32, record_mm=True)
    assert g0.stats()["tmem_cols"] == 0
    for t in range(4):
        fwd = t % 2 == 0
        g0.pass_(fwd, 0.5)
        g1.pass_(fwd, 0.5)
        assert np.array_equal(g0.lam(), g1.lam()) and np.array_equal(g0.deferred(), g1.deferred()), f"pass {t}"
        for a, b in zip(g0.min_marginals(), g1.min_marginals()):
            assert np.array_equal(a, b)
        assert _same_bound(g0, g1)
    g0.iterate(5, 0.5)
    g1.iterate(5, 0.5)
    assert np.array_equal(g0.lam(), g1.lam()) and _same_bound(g0, g1)


@pytest.mark.parametrize("name,make", [
    ("mrf", lambda: synth.mrf_potts(17, H=12, W=14, L=4)),
    ("mrf_cut", lambda: synth.mrf_potts_cut(17, H=12, W=14, L=4)),
    ("gm", lambda: synth.gm_worms_like(17, n_src=80, k_cand=6, knn=8)),
])
def test_elld_averaging(oracle_mod, monkeypatch, name, make):
    """Averaging of frequent degrees 5..32 in column-major ELL-D groups (one
    thread per variable, slots summed in ascending j -- the oracle's order, A1):
    fp64 pass by pass against the oracle at 1e-9 (lambda, delta_bar,
    min-marginals, bound), then the primal rounding (its classify / perturb
    kernel walks the same groups): a feasible labeling, objective >= LB."""
    monkeypatch.setenv("FDOG_ELLD_MIN", "1")
    monkeypatch.setenv("FDOG_FUSED", "0")
    p = make()
    g, o = _compare_pass_by_pass(p, oracle_mod, passes=4)
    lb = g.lower_bound()
    try:
        x, rounds, obj = g.round_primal(max_rounds=100)
    except F.FastdogError as e:  # no consensus within max_rounds (allowed by Alg. 2)
        assert e.code == 8
        return
    for j in range(p.n_cons):
        v, c, rel, rhs = p.row(j)
        s = int(np.dot(c, x[v]))
        assert (s <= rhs) if rel < 0 else (s >= rhs) if rel > 0 else (s == rhs)
    assert obj >= lb - 1e-6 * (1 + abs(lb))


def test_device_memory_from_torch():
    """fdog_options::dev_alloc: the solver's device memory comes from torch's
    caching allocator (the binding's default), results bit-identical to the
    library's own cudaMalloc, and destroy hands it back."""
    import gc
    import torch
    p = synth.gm_worms_like(5, n_src=60, k_cand=6, knn=6)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    g1 = F.Solver(p, precision=32)                      # allocator="torch"
    held = torch.cuda.memory_allocated() - before
    assert held >= g1.stats()["device_bytes"] > 0
    g2 = F.Solver(p, precision=32, allocator="cuda")
    assert torch.cuda.memory_allocated() - before == held
    for s in (g1, g2):
        s.iterate(5, 0.5)
    assert np.array_equal(g1.lam(), g2.lam()) and g1.lower_bound() == g2.lower_bound()
    g1.close(); g2.close()
    gc.collect()
    assert torch.cuda.memory_allocated() == before
    with pytest.raises(ValueError):
        F.Solver(p, allocator="numpy")


@pytest.mark.parametrize("mode", ["rc", "tma"])
@pytest.mark.parametrize("name,make", [
    ("gm", lambda: synth.gm_worms_like(23, n_src=60, k_cand=6, knn=6)),
    ("ct", lambda: synth.celltrack(23, frames=4, dets=40)),
    ("cut", lambda: synth.mrf_potts_cut(23, H=8, W=10, L=3)),
    ("qap", lambda: synth.qap(23, 7)),
])
def test_records_global_bitwise(oracle_mod, monkeypatch, mode, name, make):
    """Hop records read from global memory (tile kind bit 6, FDOG_RECS=global)
    instead of the stage give bit-identical iterates and bounds; one of them
    against the oracle (fp64)."""
    p = make()
    monkeypatch.setenv("FDOG_SWEEP", mode)
    monkeypatch.setenv("FDOG_FUSED", "0")
    gs = []
    for rg in ("", "global"):
        monkeypatch.setenv("FDOG_RECS", rg)
        gs.append(F.Solver(p, precision=64))
    o = oracle_mod.Oracle(p)
    s = _s(p)
    for t in range(4):
        fwd = t % 2 == 0
        for g in gs:
            g.pass_(fwd, 0.5)
        o.pass_(fwd, 0.5)
        assert np.array_equal(gs[0].lam(), gs[1].lam()) and np.array_equal(gs[0].deferred(), gs[1].deferred())
        assert gs[0].lower_bound() == gs[1].lower_bound()
        assert np.max(np.abs(gs[1].lam() - o.lam())) <= 1e-9 * s
    gs[0].iterate(3, 0.5)
    gs[1].iterate(3, 0.5)
    assert np.array_equal(gs[0].lam(), gs[1].lam()) and gs[0].lower_bound() == gs[1].lower_bound()


def test_torch_memory_reused_across_solvers():
    """A destroyed solver's device memory goes back to torch's cache and serves
    the next solver (no new cudaMalloc: torch's reserved memory stays flat),
    with identical results."""
    import gc
    import torch
    p = synth.gm_worms_like(6, n_src=80, k_cand=6, knn=6)
    pl = F.Plan(p, precision=32)
    g = F.Solver(plan=pl, precision=32)
    g.iterate(3, 0.5)
    ref = g.lam()
    g.close()
    gc.collect()
    reserved = torch.cuda.memory_reserved()
    for _ in range(3):
        h = F.Solver(plan=pl, precision=32)
        h.iterate(3, 0.5)
        assert np.array_equal(h.lam(), ref)
        h.close()
        assert torch.cuda.memory_reserved() == reserved
