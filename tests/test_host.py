"""Host-side product checks that need no GPU (-m "not gpu").

* the C-ABI library loads and exports every symbol include/fastdog.h declares;
* compiler B (product, plan.cpp) vs brute force and vs the oracle's compiler A:
  path sets, per-partition node counts bit-exact (BJ: "node and arc counts
  bit-exact"), closed forms;
* sharder / shared-variable index invariants for world > 1.
"""
import os
import re

import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth
from tests import bruteforce as bf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    hdr = open(os.path.join(ROOT, "include", "fastdog.h")).read()
    declared = set(re.findall(r"\b(fdog_[a-z_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = F.load()
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in fastdog.h but not exported"
    assert set(F.EXPORTS) == declared
    assert lib.fdog_version() >= 1


def _paths(hs, lo, hi):
    k = len(hs) - 1
    out = []

    def rec(v, h, bits):
        for beta, w in ((0, lo[v]), (1, hi[v])):
            if w == -1:
                continue
            if h == k - 1:
                if w == -2:
                    out.append(tuple(bits + [beta]))
                continue
            assert hs[h + 1] <= w < hs[h + 2]
            rec(w, h + 1, bits + [beta])

    rec(0, 0, [])
    return out


def test_compiler_b_path_sets_random_rows():
    """Compiler B: paths == brute-force X_j, canonical, P_1 = {r}."""
    rng = np.random.default_rng(77)
    done = 0
    while done < 400:
        k = int(rng.integers(1, 11))
        a = rng.integers(-5, 6, size=k)
        a[a == 0] = -2
        rel = int(rng.choice([-1, 0, 1]))
        b = int(rng.integers(-6, 7))
        X = bf.feasible_set(a, rel, b)
        p = synth.from_rows(k, np.zeros(k), [(np.arange(k), a, rel, b)])
        if X.shape[0] == 0:
            with pytest.raises(F.FastdogError) as e:
                F.Plan(p)
            assert e.value.code == 2
            continue
        hs, lo, hi = F.Plan(p).bdd(0)
        paths = _paths(hs, lo, hi)
        assert len(paths) == len(set(paths)) and set(paths) == set(map(tuple, X.tolist()))
        for h in range(k):
            sig = [(lo[v], hi[v]) for v in range(hs[h], hs[h + 1])]
            assert len(sig) == len(set(sig)) and (-1, -1) not in sig
        assert hs[1] == 1
        done += 1


def _per_hop_counts_equal(problem, oracle_mod):
    pl = F.Plan(problem)
    o = oracle_mod.Oracle(problem)
    st = pl.stats()
    assert st["nodes"] == o.total_nodes()
    assert st["arcs"] == 2 * o.total_nodes()
    for j in range(problem.n_cons):
        hs, _, _ = pl.bdd(j)
        assert np.array_equal(np.diff(hs), o.hop_widths(j)), f"row {j}"
    return st


@pytest.mark.parametrize("seed", range(30))
def test_node_counts_random_ilp(oracle_mod, seed):
    _per_hop_counts_equal(synth.random_ilp(seed, n=14, m=10, kmax=10, coef=4, forced_ok=True), oracle_mod)


@pytest.mark.parametrize("name,make", [
    ("lap4", lambda: synth.lap(synth.LAP4_LITERAL)),
    ("gm_small", lambda: synth.gm_worms_like(1, n_src=40, k_cand=5, knn=6)),
    ("mrf_small", lambda: synth.mrf_potts(1, H=6, W=7, L=3)),
    ("mrf_cut_small", lambda: synth.mrf_potts_cut(1, H=6, W=7, L=3)),
    ("gap_small", lambda: synth.gap(1, jobs=40, agents=5)),
    ("mckp_small", lambda: synth.mckp(1, classes=200, knaps=12, k=20)),
    ("qap_small", lambda: synth.qap(1, n=6)),
    ("celltrack_small", lambda: synth.celltrack(1, frames=4, dets=30)),
])
def test_node_counts_workload_shapes(oracle_mod, name, make):
    """Per-partition node counts of compiler B == compiler A (bit-exact, BJ)."""
    st = _per_hop_counts_equal(make(), oracle_mod)
    assert st["bdds"] > 0


def test_closed_forms_product():
    for k in (2, 5, 11, 50):
        p = synth.from_rows(k, np.zeros(k), [(np.arange(k), np.ones(k), 0, 1)])
        assert F.Plan(p).stats()["nodes"] == 2 * k - 1
        c = np.ones(k); c[0] = -1
        p = synth.from_rows(k, np.zeros(k), [(np.arange(k), c, 0, 0)])
        assert F.Plan(p).stats()["nodes"] == 2 * k - 1


def test_mrf_full_size_counts():
    """MRF 300x400x8 closed form: simplex rows 2*8-1, marginalisation rows 2*9-1."""
    H, W, L = 30, 40, 8   # scaled grid, same per-row shapes as the BJ config
    p = synth.mrf_potts(0, H=H, W=W, L=L)
    st = F.Plan(p).stats()
    E = H * (W - 1) + (H - 1) * W + 2 * (H - 1) * (W - 1)
    assert st["bdds"] == H * W + 2 * L * E
    assert st["nodes"] == H * W * (2 * L - 1) + 2 * L * E * (2 * (L + 1) - 1)
    assert st["shapes"] == 2


def test_mrf_potts_cut_counts():
    """Potts-cut closed form: simplex rows 2L-1 nodes, every
    3-variable cut row x_il - x_jl - z_e <= 0 has 5 nodes (partitions 1, 2, 2)."""
    H, W, L = 30, 40, 8
    p = synth.mrf_potts_cut(0, H=H, W=W, L=L)
    st = F.Plan(p).stats()
    E = H * (W - 1) + (H - 1) * W + 2 * (H - 1) * (W - 1)
    assert p.n_vars == H * W * L + E
    assert st["bdds"] == H * W + 2 * L * E
    assert st["nodes"] == H * W * (2 * L - 1) + 2 * L * E * 5
    assert st["slots"] == H * W * L + 2 * L * E * 3


def test_cooperative_tiles():
    """Shapes with a partition wider than 32 nodes (knapsack rows) become one-BDD
    cooperative tiles (kind bit 5, L = 1) with 32-bit child codes: a BDD over
    65 534 nodes is packed (the 16-bit limit applies to the lane tiles only)."""
    p = synth.gap(0, jobs=300, agents=20)
    pl = F.Plan(p)
    t = pl.tiles()
    coop = t[(t[:, 0] & 32) != 0]
    assert len(coop) == 20 and np.all(coop[:, 2] == 1) and np.all(coop[:, 3] == 1)
    assert coop[:, 4].max() > 65534
    assert pl.stats()["sweep_recompute"] == 0
    hs, lo, hi = pl.bdd(300)  # the first capacity row
    assert hs[-1] == coop[:, 4].max() or hs[-1] in set(coop[:, 4].tolist())


def test_invalid_inputs():
    base = synth.spec_two_constraint()
    bad = synth.Problem(base.n_vars, base.cost, base.row_ptr, base.col_var.copy(), base.col_coef.copy(),
                        base.rel, base.rhs)
    bad.col_coef[0] = 0
    with pytest.raises(F.FastdogError) as e:
        F.Plan(bad)
    assert e.value.code == 1
    bad = synth.Problem(base.n_vars, base.cost, base.row_ptr, base.col_var[::-1].copy(), base.col_coef,
                        base.rel, base.rhs)
    with pytest.raises(F.FastdogError):
        F.Plan(bad)
    # empty problem and free variables are fine
    p = synth.from_rows(3, [-1.0, 2.0, -0.5], [])
    st = F.Plan(p).stats()
    assert st["bdds"] == 0 and st["free_vars"] == 3


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharder_and_shared_index(world):
    """Every row on exactly one rank; the exchange list is identical on all ranks
    and equals the variables touched by rows of >= 2 ranks; local degrees sum to
    the global |J_i|."""
    p = synth.gm_worms_like(2, n_src=60, k_cand=5, knn=6)
    plans = [F.Plan(p, rank=r, world=world) for r in range(world)]
    owner = plans[0].owner()
    for pl in plans[1:]:
        assert np.array_equal(pl.owner(), owner)
    assert owner.min() >= 0 and owner.max() < world
    bdds = [pl.stats()["bdds"] for pl in plans]
    assert sum(bdds) == p.n_cons
    sv = plans[0].shared_vars()
    for pl in plans[1:]:
        assert np.array_equal(pl.shared_vars(), sv)
    ranks_of = [set() for _ in range(p.n_vars)]
    for j in range(p.n_cons):
        for i in p.row(j)[0]:
            ranks_of[i].add(int(owner[j]))
    expect = [i for i in range(p.n_vars) if len(ranks_of[i]) >= 2]
    assert list(sv) == expect
    deg = np.bincount(p.col_var, minlength=p.n_vars)
    loc = np.zeros(p.n_vars, np.int64)
    for r in range(world):
        rows = np.flatnonzero(owner == r)
        for j in rows:
            loc[p.row(j)[0]] += 1
    assert np.array_equal(loc, deg)
    # balance by BDD node count (the plan's own per-rank node totals)
    nodes = np.array([pl.stats()["nodes"] for pl in plans])
    assert nodes.max() <= 1.1 * nodes.mean() + 64
    # bundles: a variable held by exactly two rows never crosses ranks unless
    # its bundle was dissolved (none is, at this size)
    two = np.flatnonzero(deg == 2)
    assert not np.isin(two, sv).any()


def _rows_of_vars(p):
    rows = np.repeat(np.arange(p.n_cons), np.diff(p.row_ptr))
    return rows


@pytest.mark.parametrize("name,limit", [("mrf_potts", 25_000), ("qap50", 2_500), ("celltrack", 150_000),
                                        ("gm_worms_like", 6_000)])
def test_world8_exchange_volume(name, limit):
    """Locality-aware sharding at world 8 on the full-size workloads (SURVEY
    §8(e)): only the variables that cross a cut are exchanged -- MRF boundary
    pixels (~7 x 400 x 8), QAP's assignment variables (2,500), cell-tracking
    transitions across a frame cut, graph matching's x (5.5k) -- and every rank
    holds 1/8 of the BDD nodes within 2 %.  The exchange vector is the set of
    variables touched by rows of >= 2 ranks, recomputed here from the owner map."""
    p = synth.WORKLOADS[name](0)
    pl = F.Plan(p, rank=0, world=8)
    owner = pl.owner()
    sv = pl.shared_vars()
    assert sv.size <= limit, (name, sv.size)
    rows = _rows_of_vars(p)
    r = owner[rows].astype(np.int64)
    lo = np.full(p.n_vars, 99, np.int64)
    hi = np.full(p.n_vars, -1, np.int64)
    np.minimum.at(lo, p.col_var, r)
    np.maximum.at(hi, p.col_var, r)
    assert np.array_equal(np.flatnonzero((hi >= 0) & (lo != hi)), sv)
    k = np.diff(p.row_ptr)
    w = np.zeros(8)
    np.add.at(w, owner, k)  # nnz per rank (nodes ~ 2k - 1 for these row families)
    assert w.max() <= 1.02 * w.mean(), w


def test_row_owner_option():
    """A caller-supplied row -> rank map replaces the sharder (fdog_options.row_owner)."""
    p = synth.gm_worms_like(2, n_src=40, k_cand=4, knn=5)
    own = (np.arange(p.n_cons) % 3).astype(np.int32)
    pls = [F.Plan(p, rank=r, world=3, row_owner=own) for r in range(3)]
    assert np.array_equal(pls[0].owner(), own)
    assert sum(pl.stats()["bdds"] for pl in pls) == p.n_cons
    bad = own.copy()
    bad[0] = 3
    with pytest.raises(F.FastdogError):
        F.Plan(p, rank=0, world=3, row_owner=bad)


def _pattern(hs, lo, hi, h):
    """Arc targets of partition h: per node (lo, hi) as 'next j' / 'T' / 'B'."""
    n1 = hs[h + 1]
    out = []
    for n in range(hs[h], n1):
        out.append(tuple("B" if c == -1 else "T" if c == -2 else int(c - n1) for c in (lo[n], hi[n])))
    return out


@pytest.mark.parametrize("name,make", [
    ("gm", lambda: synth.gm_worms_like(3, n_src=60, k_cand=5, knn=6)),
    ("mrf", lambda: synth.mrf_potts(3, H=8, W=9, L=4)),
    ("qap", lambda: synth.qap(3, n=7)),
    ("ct", lambda: synth.celltrack(3, frames=4, dets=30)),
    ("thin", lambda: synth.thin_hop(3, k=2000)),  # too long to stage: a partly filled records tile
])
def test_hop_record_classes(name, make):
    """Tile kind bits the kernels rely on, re-derived from each row's compiled
    BDD: arc-mask tiles (bit 2) have partitions of <= 2 nodes; chain tiles
    (bit 3) have the chain pattern 0->0, 1->1 (0-arcs), 1->0 (1-arc) in every
    middle partition; root/join tiles (bit 4) have a one-node root with arcs
    to nodes 0 / 1, partition sizes 1, 2, ..., 2 (node indices 2h-1, 2h: the
    folded kernels compute them) and a last partition joining into top."""
    p = make()
    pl = F.Plan(p, precision=32)
    tiles = pl.tiles()
    smap = pl.slot_map()
    nonempty = np.diff(p.row_ptr) > 0
    first = {int(smap[p.row_ptr[j]]): j for j in range(p.n_cons) if nonempty[j]}
    seen = 0
    for kind, K, L, nl, nodes, base in tiles:
        if not kind & 4:
            assert not kind & 24
            continue
        for lane in range(nl):
            j = first[int(base + lane)]
            hs, lo, hi = pl.bdd(j)
            assert len(hs) - 1 == K and np.all(np.diff(hs) <= 2)
            if kind & 8:
                for h in range(1, K - 1):
                    assert _pattern(hs, lo, hi, h) == [(0, "B"), (1, 0)], (name, j, h)
            if kind & 16:
                assert kind & 8 and K >= 2
                assert list(np.diff(hs)) == [1] + [2] * (K - 1) and hs[-1] == 2 * K - 1 == nodes
                assert _pattern(hs, lo, hi, 0) == [(0, 1)]
                assert _pattern(hs, lo, hi, K - 1) == [("T", "B"), ("B", "T")]
            seen += 1
    assert seen > 0


@pytest.mark.parametrize("name,make", [
    ("gm", lambda: synth.gm_worms_like(5)),                 # 2.3 M slots: many 64 K chunks
    ("mrf", lambda: synth.mrf_potts(5, H=60, W=80, L=8)),
    ("ct", lambda: synth.celltrack(5, frames=30, dets=600)),
    ("wide", lambda: synth.random_ilp(5, n=60, m=200, kmax=10, coef=4)),
])
def test_plan_deterministic_across_threads(name, make):
    """The parallel packing phases (chunks of 64 K items) give byte-identical
    plans -- every packed array and the device image -- for 1, 3 and 8 host
    threads."""
    p = make()
    d = {t: F.Plan(p, precision=32, host_threads=t).digest() for t in (1, 3, 8)}
    assert d[1] == d[3] == d[8]
    assert F.Plan(p, precision=64, host_threads=1).digest() == F.Plan(p, precision=64, host_threads=8).digest()


def test_lifted_plan_layout():
    """Lifted plans (fdog_options::lifted): every tile unstaged (the
    sweeps read both arc costs from global memory), no arc-mask records, no
    rows-per-lane or tile-closed pairs, no recompute design; world 1 only."""
    p = synth.mrf_potts(2, H=12, W=12, L=4)
    pl = F.Plan(p, lifted=True)
    t = pl.tiles()
    st = pl.stats()
    assert np.all((t[:, 0] & (2 | 4)) == 0) and t[:, 2].max() <= 32
    assert st["staged_tiles"] == 0 and st["tile_pairs"] == 0 and st["sweep_recompute"] == 0
    with pytest.raises(F.FastdogError) as e:
        F.Plan(p, world=2, lifted=True)
    assert e.value.code == 1
