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


def _gather(p, ranks, oracle_n):
    lam = np.full(oracle_n, np.nan)
    dl = np.full(oracle_n, np.nan)
    for g in ranks:
        con, pos = g.slot_index()
        idx = p.row_ptr[con] + pos
        lam[idx] = g.lam()
        dl[idx] = g.deferred()
    return lam, dl


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,make", [
    ("gm", lambda: synth.gm_worms_like(13, n_src=60, k_cand=6, knn=6)),
    ("mrf", lambda: synth.mrf_potts(13, H=10, W=12, L=4)),
])
def test_peer_exchange_equals_host_exchange(oracle_mod, precision, world, name, make):
    """Peer-memory exchange (fdog_set_peer_regions; the regions as plain device
    pointers, one process): after every pass bit-identical to the host-summed
    exchange in rank order, and within 1e-9 of the oracle (fp64)."""
    p = make()
    s = max(1.0, float(np.abs(p.cost).max()))
    host = [F.Solver(p, precision=precision, rank=r, world=world) for r in range(world)]
    peer = [F.Solver(p, precision=precision, rank=r, world=world) for r in range(world)]
    regions = [g.exchange_region()[0] for g in peer]
    for g in peer:
        g.set_peer_regions(regions)
    o = oracle_mod.Oracle(p)
    for t in range(6):
        fwd = t % 2 == 0
        for g in host:
            g.pass_begin(fwd, 0.5)
        # rank order, in the solver's precision, as the device sums
        dt = np.float64 if precision == 64 else np.float32
        x = np.zeros(1, dt)
        for g in host:
            x = (x + g.exchange_read().astype(dt)).astype(dt)
        x = x.astype(np.float64)
        for g in host:
            g.exchange_write(x)
        for g in host:
            g.pass_end(fwd, 0.5)
        for g in peer:      # every rank publishes ...
            g.pass_begin(fwd, 0.5)
        for g in peer:      # ... before any waits (one thread drives all ranks)
            g.pass_end(fwd, 0.5)
        o.pass_(fwd, 0.5)
        for a, b in zip(host, peer):
            assert np.array_equal(a.lam(), b.lam()) and np.array_equal(a.deferred(), b.deferred()), f"pass {t}"
        if precision == 64:
            lam, dl = _gather(p, peer, o.num_slots())
            assert np.max(np.abs(lam - o.lam())) <= 1e-9 * s, f"pass {t}"
            assert np.max(np.abs(dl - o.deferred())) <= 1e-9 * s
    assert all(g.peer_error() == 0 for g in peer)


def test_peer_exchange_whole_passes_on_streams(oracle_mod):
    """fdog_iterate in the peer mode: each rank's whole pass on its own stream,
    launched one rank after the other from one thread -- the ranks wait for
    each other on the device only."""
    import torch
    p = synth.gm_worms_like(14, n_src=60, k_cand=6, knn=6)
    s = max(1.0, float(np.abs(p.cost).max()))
    world = 2
    streams = [torch.cuda.Stream() for _ in range(world)]
    ranks = [F.Solver(p, precision=64, rank=r, world=world, stream=streams[r].cuda_stream) for r in range(world)]
    regions = [g.exchange_region()[0] for g in ranks]
    for g in ranks:
        g.set_peer_regions(regions, timeout_s=10.0)
    o = oracle_mod.Oracle(p)
    for it in range(3):
        for g in ranks:
            g.iterate(1, 0.5)
        o.iterate(1, 0.5)
        assert all(g.peer_error() == 0 for g in ranks)
        lam, dl = _gather(p, ranks, o.num_slots())
        assert np.max(np.abs(lam - o.lam())) <= 1e-9 * s, it
        lb = sum(g.lower_bound() for g in ranks)
        assert abs(lb - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
    # averaged final correction (A11 prose reading) through the peer exchange
    for g in ranks:
        g.finalize(averaged=True)
    o.finalize(averaged=True)
    assert all(g.peer_error() == 0 for g in ranks)
    lam, dl = _gather(p, ranks, o.num_slots())
    assert np.max(np.abs(lam - o.lam())) <= 1e-9 * s
    assert np.all(dl == 0.0)
    lb = sum(g.lower_bound() for g in ranks)
    assert abs(lb - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)


def test_peer_exchange_errors_and_timeout():
    p = synth.gm_worms_like(15, n_src=40, k_cand=5, knn=5)
    single = F.Solver(p, precision=32)
    with pytest.raises(F.FastdogError) as e:
        single.exchange_region()
    assert e.value.code == 6
    ranks = [F.Solver(p, precision=32, rank=r, world=2) for r in range(2)]
    regions = [g.exchange_region()[0] for g in ranks]
    with pytest.raises(F.FastdogError) as e:
        ranks[0].set_peer_regions(regions[:1])          # wrong world size
    assert e.value.code == 1
    with pytest.raises(F.FastdogError) as e:
        ranks[0].set_peer_regions(regions[::-1])        # own region not at [rank]
    assert e.value.code == 1
    ranks[0].set_peer_regions(regions, timeout_s=0.2)
    ranks[0].pass_(True, 0.5)                           # rank 1 never publishes
    assert ranks[0].peer_error() == 1                   # reported, no hang
    ranks[1].pass_begin(True, 0.5)
    ranks[1].pass_end(True, 0.5)
    with pytest.raises(F.FastdogError) as e:
        ranks[1].set_peer_regions(regions)              # after a pass
    assert e.value.code == 6


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("name,make", [
    ("gm", lambda: synth.gm_worms_like(14, n_src=80, k_cand=6, knn=8)),
    ("mrf", lambda: synth.mrf_potts(14, H=16, W=18, L=4)),
])
def test_nccl_graph_overlap_one_gpu(monkeypatch, precision, name, make):
    """The NCCL path of a world-2 rank on one GPU (FDOG_NCCL_SELF=1: a one-rank
    communicator, so ncclAllReduce is the identity on this rank's partials):
    fdog_iterate captures the whole iteration -- averaging, the exchange forked
    onto a second stream (ncclAllReduce + avg_finish), the interior tiles'
    sweep overlapping it, the boundary tiles' sweep after the join -- into one
    CUDA graph.  Bit for bit equal to (a) the same solver with direct launches
    and the exchange run first (FDOG_GRAPHS=0, FDOG_OVERLAP=0) and (b) the
    external-exchange mode where the test writes each rank's own partials back
    (the identity exchange, host-driven)."""
    import os
    import torch
    import nvidia.nccl
    lib = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
    p = make()
    monkeypatch.setenv("FDOG_NCCL_SELF", "1")
    g = F.Solver(p, precision=precision, rank=0, world=2, nccl_unique_id=torch.cuda.nccl.unique_id(),
                 nccl_library=lib)
    st = g.stats()
    assert 0 < st["vars_shared"] and 0 < st["interior_tiles"] < st["tiles"]
    monkeypatch.setenv("FDOG_GRAPHS", "0")
    monkeypatch.setenv("FDOG_OVERLAP", "0")
    d = F.Solver(p, precision=precision, rank=0, world=2, nccl_unique_id=torch.cuda.nccl.unique_id(),
                 nccl_library=lib)
    monkeypatch.delenv("FDOG_GRAPHS")
    monkeypatch.delenv("FDOG_OVERLAP")
    monkeypatch.delenv("FDOG_NCCL_SELF")
    h = F.Solver(p, precision=precision, rank=0, world=2)  # external exchange
    for it in range(4):
        g.iterate(1, 0.5)
        d.iterate(1, 0.5)
        for fwd in (True, False):
            h.pass_begin(fwd, 0.5)
            h.exchange_write(h.exchange_read())
            h.pass_end(fwd, 0.5)
        assert np.array_equal(g.lam(), d.lam()) and np.array_equal(g.lam(), h.lam()), f"iteration {it}"
        assert np.array_equal(g.deferred(), h.deferred())
    g.close()
    d.close()
