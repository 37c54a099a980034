"""compute-sanitizer case for the last kernels of round 1: single/double-buffered
store-design stages, the early PDL release, the CSR-first averaging with index
prefetch, and the peer-memory exchange (two ranks in one process, driven by
pass_begin for every rank before any pass_end: the sanitizer serialises
kernels, so no rank may wait on a peer that has not been launched)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2111_10270_b200 as F
probs = (synth.gm_worms_like(3, n_src=40, k_cand=4, knn=4), synth.celltrack(3, frames=3, dets=20),
         synth.mrf_potts(3, H=5, W=6, L=3))
os.environ["FDOG_SWEEP"] = "tma"
os.environ["FDOG_FUSED"] = "0"
for nb in ("1", "2"):
    for early in ("0", "1"):
        os.environ["FDOG_NBUF"] = nb
        os.environ["FDOG_PDL_EARLY"] = early
        for p in probs:
            for prec in (32, 64):
                s = F.Solver(p, precision=prec)
                s.iterate(3, 0.5); s.pass_(True, 0.5)
                s.lower_bound(); s.lam(); s.close()
for k in ("FDOG_SWEEP", "FDOG_FUSED", "FDOG_NBUF", "FDOG_PDL_EARLY"):
    os.environ.pop(k)
for p in probs:
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
            g.lower_bound(); g.lam(); g.close()
print("sanitize case 3 ok")
