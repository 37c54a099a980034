"""Peer-memory exchange across processes (one process per rank, as on a
multi-GPU node): each rank maps the others' exchange regions through CUDA IPC
(fdog_ipc_handle / fdog_ipc_open) and runs whole iterations with no host
exchange.  Here both processes share the one GPU (contexts time-slice); on a
node each has its own GPU and the loads go over NVLink.  Checked against the
unsharded fp64 oracle."""
import multiprocessing as mp

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

WORLD = 2


def _problem():
    return synth.gm_worms_like(16, n_src=60, k_cand=6, knn=6)


def _worker(rank, conn):
    import paper_2111_10270_b200 as F
    p = _problem()
    g = F.Solver(p, precision=64, rank=rank, world=WORLD)
    own, _ = g.exchange_region()
    conn.send(F.ipc_handle(own))
    handles = conn.recv()
    regions = [own if k == rank else F.ipc_open(h) for k, h in enumerate(handles)]
    g.set_peer_regions(regions, timeout_s=30.0)
    g.iterate(2, 0.5)
    con, pos = g.slot_index()
    conn.send((g.peer_error(), con, pos, g.lam(), g.lower_bound()))
    conn.recv()  # every rank has finished reading the others' regions
    for k, r in enumerate(regions):
        if k != rank:
            F.ipc_close(r)
    g.close()


def test_peer_exchange_across_processes(oracle_mod):
    ctx = mp.get_context("spawn")
    pipes = [ctx.Pipe() for _ in range(WORLD)]
    procs = [ctx.Process(target=_worker, args=(r, pipes[r][1])) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    try:
        conns = [a for a, _ in pipes]
        for c in conns:
            assert c.poll(300), "worker did not start"
        handles = [c.recv() for c in conns]
        for c in conns:
            c.send(handles)
        res = []
        for c in conns:
            assert c.poll(300), "worker did not finish"
            res.append(c.recv())
        for c in conns:
            c.send("done")
    finally:
        for pr in procs:
            pr.join(60)
            if pr.is_alive():
                pr.kill()
    assert all(pr.exitcode == 0 for pr in procs)
    p = _problem()
    o = oracle_mod.Oracle(p)
    o.iterate(2, 0.5)
    s = max(1.0, float(np.abs(p.cost).max()))
    lam = np.full(o.num_slots(), np.nan)
    for err, con, pos, l_, lb in res:
        assert err == 0
        lam[p.row_ptr[con] + pos] = l_
    assert not np.isnan(lam).any()
    assert np.max(np.abs(lam - o.lam())) <= 1e-9 * s
    assert abs(sum(r[4] for r in res) - o.lower_bound()) <= 1e-9 * (abs(o.lower_bound()) + s)
