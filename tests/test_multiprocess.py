"""World-size-2 (and 3) CPU tests of the multi-GPU host path with torch.distributed/gloo.

Each rank builds its own plan (product sharder, plan.cpp) exactly as bench.py's
torchrun ranks do.  Checked across ranks through real collectives:
  * every rank derives the same row->rank map and the same exchange vector;
  * the deferred averaging decomposes over ranks: per-rank
    partial sums over the rank's own slots, summed by all_reduce and divided by
    the global |J_i|, reproduce the unsharded average of the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2111_10270_b200 as F
    import synth
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p = synth.gm_worms_like(11, n_src=50, k_cand=5, knn=6)
        plan = F.Plan(p, rank=rank, world=world)
        owner = plan.owner()
        shared = plan.shared_vars()
        # identical maps on every rank
        for arr in (torch.from_numpy(owner.astype(np.int64)), torch.from_numpy(shared.astype(np.int64))):
            gathered = [torch.empty_like(arr) for _ in range(world)]
            dist.all_gather(gathered, arr)
            assert all(torch.equal(g, arr) for g in gathered)
        # a few oracle passes give a realistic delta_bar (canonical slots)
        o = oracle.Oracle(p, n_threads=1)
        o.iterate(2, 0.5)
        o.pass_(True, 0.5)
        delta = o.deferred()
        row_of_slot = np.repeat(np.arange(p.n_cons), np.diff(p.row_ptr))
        mine = owner[row_of_slot] == rank
        partial = np.zeros(p.n_vars)
        np.add.at(partial, p.col_var[mine], delta[mine])
        # exchange only the shared variables (the product's xbuf), sum over ranks
        x = torch.from_numpy(partial[shared].copy())
        dist.all_reduce(x)
        deg = np.bincount(p.col_var, minlength=p.n_vars)
        avg = np.where(deg > 0, partial / np.maximum(deg, 1), 0.0)
        avg[shared] = x.numpy() / deg[shared]
        # unsharded reference average
        full = np.zeros(p.n_vars)
        np.add.at(full, p.col_var, delta)
        ref = np.where(deg > 0, full / np.maximum(deg, 1), 0.0)
        used = np.zeros(p.n_vars, bool)
        used[p.col_var[mine]] = True  # variables this rank needs
        assert np.allclose(avg[used], ref[used], rtol=1e-12, atol=1e-12)
        # variables not in the exchange vector are held by this rank alone
        not_shared = np.setdiff1d(np.flatnonzero(used), shared)
        others = np.zeros(p.n_vars, bool)
        others[p.col_var[~mine]] = True
        assert not others[not_shared].any()
        st = plan.stats()
        n = torch.tensor([st["bdds"], st["nodes"]], dtype=torch.int64)
        dist.all_reduce(n)
        q.put((rank, "ok", int(n[0]), int(n[1])))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e), 0, 0))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_plans_and_exchange_gloo(world, oracle_mod):
    import paper_2111_10270_b200 as F
    import synth
    F.load()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, msg, _, _ in res:
        assert msg == "ok", f"rank {rank}: {msg}"
    p = synth.gm_worms_like(11, n_src=50, k_cand=5, knn=6)
    full = F.Plan(p).stats()
    assert res[0][2] == full["bdds"] and res[0][3] == full["nodes"]
