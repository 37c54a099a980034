"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration
(fp32, the design the plan picks, CUDA-graph replay for iterate), for the
workloads besides GM (GM: test_gpu_parity.py::test_full_size_gm_*).

- CellTrack (configs[3], 9.7 M nodes), QAP n=50 (configs[4], 12.1 M nodes) and
  the MRF Potts-cut variant (40.0 M nodes; rows per lane, ELL-D averaging):
  every slot of lambda after one iteration against the oracle (fp64), the
  bound after 100 iterations (north_star's fp32 claim); fp64 builds every slot
  at 1e-9 for two iterations.
- MRF Potts (configs[2], 131.8 M nodes; the bench workload): fp64 every slot of
  lambda and delta_bar plus the bound after each of two whole iterations at
  1e-9 (the oracle holds ~10 GB and runs ~1.6 s per iteration on 16 cores);
  fp32 every slot after two iterations, the bound after 20.
- MRF and QAP n=128 (the 8-GPU stress configuration, 530.7 M nodes, on one
  GPU; its oracle would need tens of GB): first passes sampled.  The first pass from the initial state has
  delta_bar = 0, so avg_i = 0 and every BDD is updated independently
  of the others; the oracle run on a sub-problem made of sampled rows,
  with costs rescaled so that the initial lambda = c_i / |J_i| is the
  full problem's, must reproduce their lambda and delta (fdog_get_deferred)
  exactly up to rounding.  Forward and backward first passes.
Tolerances: fp32 |a - b| <= 1e-5 (|b| + s), fp64 1e-9,
s = max(1, max|c|).
"""
import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth

pytestmark = pytest.mark.gpu


def _s(p):
    return max(1.0, float(np.max(np.abs(p.cost))))


def _err(a, b, rtol, s):
    return float(np.max(np.abs(a - b) - rtol * np.abs(b), initial=-1.0)) - rtol * s


@pytest.fixture(scope="module", params=["celltrack", "qap50", "mrf_potts_cut"])
def full_problem(request):
    if request.param == "celltrack":
        return synth.celltrack(0)
    if request.param == "mrf_potts_cut":  # the Potts-cut variant of the metric's MRF line (40.0 M nodes)
        return synth.mrf_potts_cut(0)
    return synth.qap(0, 50)


def test_full_size_fp32(oracle_mod, full_problem):
    p = full_problem
    g = F.Solver(p, precision=32)
    o = oracle_mod.Oracle(p)
    st = g.stats()
    assert st["nodes"] == o.total_nodes() and st["arcs"] == 2 * o.total_nodes()
    s = _s(p)
    g.iterate(1, 0.5)
    o.iterate(1, 0.5)
    assert _err(g.lam(), o.lam(), 1e-5, s) <= 0
    assert _err(g.deferred(), o.deferred(), 1e-5, s) <= 0
    g.iterate(99, 0.5)
    o.iterate(99, 0.5)
    assert abs(g.lower_bound() - o.lower_bound()) <= 1e-4 * abs(o.lower_bound())


def test_full_size_fp64(oracle_mod, full_problem):
    p = full_problem
    g = F.Solver(p, precision=64)
    o = oracle_mod.Oracle(p)
    s = _s(p)
    for _ in range(2):
        g.iterate(1, 0.5)
        o.iterate(1, 0.5)
        assert _err(g.lam(), o.lam(), 1e-9, s) <= 0
        assert abs(g.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)


def test_full_size_mrf(oracle_mod):
    """MRF Potts 300x400x8 (BASELINE configs[2], the bench workload) in bench.py's
    launch configuration: fp64 every slot of lambda and delta_bar and the bound
    after each of 2 whole iterations at 1e-9; fp32 every slot after 2 iterations
    at 1e-5 and the bound after 20 within 1e-4 relative; node/arc counts exact."""
    p = synth.mrf_potts(0)
    s = _s(p)
    o = oracle_mod.Oracle(p)
    g64 = F.Solver(p, precision=64)
    st = g64.stats()
    assert st["nodes"] == o.total_nodes() == 131_789_344 and st["arcs"] == 2 * o.total_nodes()
    for _ in range(2):
        g64.iterate(1, 0.5)
        o.iterate(1, 0.5)
        assert _err(g64.lam(), o.lam(), 1e-9, s) <= 0
        assert _err(g64.deferred(), o.deferred(), 1e-9, s) <= 0
        assert abs(g64.lower_bound() - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    g64.close()
    g32 = F.Solver(p, precision=32)
    g32.iterate(2, 0.5)
    assert _err(g32.lam(), o.lam(), 1e-5, s) <= 0
    assert _err(g32.deferred(), o.deferred(), 1e-5, s) <= 0
    g32.iterate(18, 0.5)
    o.iterate(18, 0.5)
    assert abs(g32.lower_bound() - o.lower_bound()) <= 1e-4 * abs(o.lower_bound())


def sub_problem(p, rows):
    """The sampled rows as a problem of their own (same variables), costs scaled
    by |J_i in the sample| / |J_i| so that the initial multipliers agree."""
    deg = np.bincount(p.col_var, minlength=p.n_vars).astype(float)
    rr = [p.row(int(j)) for j in rows]
    deg_s = np.zeros(p.n_vars)
    for v, c, rel, rhs in rr:
        deg_s[v] += 1
    cost = np.where(deg > 0, p.cost * deg_s / np.maximum(deg, 1), 0.0)
    return synth.from_rows(p.n_vars, cost, rr, "sample"), rr


@pytest.fixture(scope="module", params=["mrf_potts", "qap128"])
def big_problem(request):
    if request.param == "mrf_potts":
        return synth.mrf_potts(0)
    return synth.qap(0, 128)


@pytest.mark.parametrize("forward", [True, False])
def test_full_size_first_pass_sampled(oracle_mod, big_problem, forward):
    p = big_problem
    g = F.Solver(p, precision=32)
    g.pass_(forward, 0.5)
    lam, dl = g.lam(), g.deferred()
    rng = np.random.default_rng(7 + forward)
    rows = np.unique(np.concatenate([rng.choice(p.n_cons, size=400, replace=False),
                                     [0, p.n_cons - 1]]))
    sub, rr = sub_problem(p, rows)
    o = oracle_mod.Oracle(sub)
    o.pass_(forward, 0.5)
    olam, odl = o.lam(), o.deferred()
    s = _s(p)
    base = 0
    for j, (v, c, rel, rhs) in zip(rows, rr):
        a0, k = int(p.row_ptr[j]), len(v)
        assert _err(lam[a0:a0 + k], olam[base:base + k], 1e-5, s) <= 0, j
        assert _err(dl[a0:a0 + k], odl[base:base + k], 1e-5, s) <= 0, j
        base += k
    assert base == len(olam)
