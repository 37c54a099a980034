"""BDD compilation on the GPU (compile_gpu.cu) is identical to
the host compiler B: every compiled BDD (partition sizes, child codes) and the
whole packed plan (digest of every array and the device image)."""
import numpy as np
import pytest

import paper_2111_10270_b200 as F
import synth

pytestmark = pytest.mark.gpu


def _rows_wide(seed, n=40, m=120, kmax=14, coef=9):
    """Rows with large coefficients of both signs and all three relations
    (wide partitions, many distinct suffix sums)."""
    rng = np.random.default_rng(seed)
    rows = []
    while len(rows) < m:
        k = int(rng.integers(1, kmax + 1))
        v = np.sort(rng.choice(n, size=k, replace=False))
        a = rng.integers(1, coef + 1, size=k) * rng.choice([-1, 1], size=k)
        lo, hi = int(np.minimum(a, 0).sum()), int(np.maximum(a, 0).sum())
        rel = int(rng.choice([synth.LE, synth.EQ, synth.GE]))
        b = int(rng.integers(lo, hi + 1))
        xs = ((np.arange(2 ** k)[:, None] >> np.arange(k)[None, :]) & 1)
        s = xs @ a
        ok = (s <= b) if rel == synth.LE else (s >= b) if rel == synth.GE else (s == b)
        if ok.any():
            rows.append((v, a, rel, b))
    return synth.from_rows(n, rng.uniform(-1, 1, size=n), rows, f"wide({seed})")


CASES = [
    ("wide0", lambda: _rows_wide(0)),
    ("wide1", lambda: _rows_wide(1, kmax=20, coef=3)),
    ("random", lambda: synth.random_ilp(3, n=30, m=80, kmax=9, coef=5, forced_ok=True)),
    ("gm", lambda: synth.gm_worms_like(7, n_src=80, k_cand=6, knn=8)),
    ("ct", lambda: synth.celltrack(7, frames=6, dets=60)),
    ("qap", lambda: synth.qap(7, n=9)),
    ("thin", lambda: synth.thin_hop(7, k=3000)),
]


@pytest.mark.parametrize("name,make", CASES)
def test_gpu_compile_identical(monkeypatch, name, make):
    p = make()
    plans = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("FDOG_GPU_COMPILE", mode)
        plans[mode] = F.Plan(p, precision=32)
    for j in range(0, p.n_cons, max(1, p.n_cons // 300)):
        a, b = plans["0"].bdd(j), plans["1"].bdd(j)
        assert all(np.array_equal(x, y) for x, y in zip(a, b)), (name, j)
    assert plans["0"].digest() == plans["1"].digest()


def test_gpu_compile_infeasible_row(monkeypatch):
    p = synth.from_rows(3, np.zeros(3), [([0, 1, 2], [1, 1, 1], synth.GE, 4)])
    for mode in ("0", "1"):
        monkeypatch.setenv("FDOG_GPU_COMPILE", mode)
        with pytest.raises(F.FastdogError) as e:
            F.Plan(p)
        assert e.value.code == 2


@pytest.mark.parametrize("name,make", CASES + [
    ("mrf", lambda: synth.mrf_potts(7, H=20, W=24, L=4)),
    ("mrf_cut", lambda: synth.mrf_potts_cut(7, H=16, W=18, L=5)),
    ("gap", lambda: synth.gap(7, jobs=40, agents=5)),
])
@pytest.mark.parametrize("opts", [{}, {"world": 2, "rank": 1}, {"lifted": True}, {"precision": 64}])
def test_gpu_pack_identical(monkeypatch, name, make, opts):
    """The packer's canonical-slot and variable phases on the GPU
    (FDOG_GPU_PACK=1, pack_gpu.cu: scans, atomic-min first slots, a stable
    radix sort) give the host packer's plan byte for byte (digest of every
    array and the device image), for sharded, lifted and fp64 plans too."""
    if opts.get("lifted") and opts.get("world", 1) > 1:
        pytest.skip("lifted plans are single-GPU")
    p = make()
    monkeypatch.setenv("FDOG_GPU_PACK", "0")
    host = F.Plan(p, **opts).digest()
    monkeypatch.setenv("FDOG_GPU_PACK", "1")
    gpu = F.Plan(p, **opts).digest()
    assert gpu == host


def test_gpu_pack_full_mrf_digest(monkeypatch):
    """MRF-LP at full size, compiled and packed on the GPU (the default at
    this size): same digest as the host compiler and packer."""
    p = synth.mrf_potts(0)
    monkeypatch.setenv("FDOG_GPU_PACK", "1")
    monkeypatch.setenv("FDOG_GPU_COMPILE", "1")
    a = F.Plan(p).digest()
    monkeypatch.setenv("FDOG_GPU_PACK", "0")
    monkeypatch.setenv("FDOG_GPU_COMPILE", "0")
    assert a == F.Plan(p).digest()


@pytest.mark.parametrize("name,make", CASES[:3] + [("gap", lambda: synth.gap(8, jobs=40, agents=5))])
def test_gpu_compile_vs_oracle_compiler(monkeypatch, oracle_mod, name, make):
    """The GPU compiler against the oracle's independent compiler A (top-down
    partial sums, bottom-up signature merge): per-partition node counts of
    every BDD equal (the canonical quasi-reduced form is unique, A12)."""
    p = make()
    monkeypatch.setenv("FDOG_GPU_COMPILE", "1")
    pl = F.Plan(p)
    o = oracle_mod.Oracle(p)
    assert pl.stats()["nodes"] == o.total_nodes()
    for j in range(p.n_cons):
        hs, _, _ = pl.bdd(j)
        assert np.array_equal(np.diff(hs), o.hop_widths(j)), f"row {j}"
