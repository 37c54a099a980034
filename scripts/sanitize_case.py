"""compute-sanitizer target (scripts/gpu_sanitize.sh): every kernel family on
small instances -- the three sweep designs, averaging, primal rounding; the
non-deferred passes, the chunked sweep, the GPU compiler; single / double
stage buffers; the peer exchange (two ranks in one process: pass_begin for
every rank before any pass_end, the sanitizer serialises kernels); rows per
lane, wide BDDs node-parallel, TMEM distances, the lifted representation."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_10270_b200 as F  # noqa: E402
import synth  # noqa: E402


def run(p, prec, **kw):
    s = F.Solver(p, precision=prec, record_mm=True, **kw)
    s.iterate(3, 0.5)
    s.pass_(True, 0.5)
    s.pass_(False, 0.5)
    s.pass_(False, 0.5)
    s.lower_bound()
    s.min_marginals()
    s.finalize()
    s.iterate(1, 0.5)
    s.lam()
    return s


def env(**kv):
    for k, v in kv.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


small = (synth.gm_worms_like(3, n_src=40, k_cand=4, knn=4), synth.qap(3, n=6), synth.celltrack(3, frames=3, dets=20),
         synth.mrf_potts(3, H=5, W=6, L=3), synth.lap(synth.LAP4_LITERAL))
# designs, averaging, rounding
for mode in ("rc", "tma", "stream"):
    env(FDOG_SWEEP=mode)
    for p in small + ((synth.random_ilp(7, n=40, m=60, kmax=12, coef=5),) if mode == "tma" else ()):
        for prec in (32, 64):
            s = run(p, prec)
            try:
                s.round_primal(max_rounds=5)
            except F.FastdogError as e:
                assert e.code == 8
            s.close()
env(FDOG_SWEEP=None)
# non-deferred passes, chunked sweep (long rows), GPU compiler
env(FDOG_GPU_COMPILE="1")
rng = np.random.default_rng(0)
rows = [(np.sort(rng.choice(1500, size=900, replace=False)), np.ones(900), synth.LE, 1) for _ in range(3)]
rows += [(np.array([q, q + 1]), np.ones(2), synth.LE, 1) for q in range(0, 1499, 2)]
long_rows = synth.from_rows(1500, rng.uniform(-1, 1, 1500), rows, "long")
for p in (small[0], small[3], long_rows, synth.thin_hop(3, k=700)):
    for prec in (32, 64):
        s = run(p, prec)
        s.iterate_seq(2, 0.5)
        s.pass_seq(True, 0.5)
        s.close()
env(FDOG_GPU_COMPILE=None)
# stage buffers (store design)
env(FDOG_SWEEP="tma", FDOG_FUSED="0")
for nb in ("1", "2"):
    env(FDOG_NBUF=nb)
    for p in small[:4]:
        for prec in (32, 64):
            run(p, prec).close()
env(FDOG_SWEEP=None, FDOG_FUSED=None, FDOG_NBUF=None)
# rows per lane, TMEM distances
env(FDOG_FUSED="0", FDOG_WIDE="1")
for p in (synth.mrf_potts(9, H=20, W=24, L=4), synth.mrf_potts_cut(9, H=16, W=18, L=5)):
    for prec in (32, 64):
        run(p, prec).close()
env(FDOG_WIDE=None, FDOG_SWEEP="rc", FDOG_TMEM="1")
for p in (synth.qap(16, n=12), synth.celltrack(16, frames=8, dets=60)):
    run(p, 32).close()
env(FDOG_SWEEP=None, FDOG_TMEM=None, FDOG_FUSED=None)
# wide BDDs node-parallel; the lifted representation
for p in (synth.gap(1, jobs=40, agents=5), synth.mckp(1, classes=200, knaps=12, k=20)):
    for prec in (32, 64):
        run(p, prec).close()
        run(p, prec, lifted=True).close()
# peer exchange
for p in small[:4]:
    for prec in (32, 64):
        rk = [F.Solver(p, precision=prec, rank=r, world=2) for r in range(2)]
        regs = [g.exchange_region()[0] for g in rk]
        for g in rk:
            g.set_peer_regions(regs, timeout_s=60.0)
        for t in range(4):
            for g in rk:
                g.pass_begin(t % 2 == 0, 0.5)
            for g in rk:
                g.pass_end(t % 2 == 0, 0.5)
        assert all(g.peer_error() == 0 for g in rk)
        for g in rk:
            g.lower_bound()
            g.close()
print("sanitize case ok")
