"""Small end-to-end GPU run for compute-sanitizer: all three sweep designs, averaging, rounding."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2111_10270_b200 as F
for mode in ("rc", "tma", "stream"):
    os.environ["FDOG_SWEEP"] = mode
    for p in (synth.gm_worms_like(3, n_src=40, k_cand=4, knn=4), synth.qap(3, n=6),
              synth.random_ilp(7, n=40, m=60, kmax=12, coef=5) if mode == "tma" else synth.lap(synth.LAP4_LITERAL),
              synth.celltrack(3, frames=3, dets=20), synth.mrf_potts(3, H=5, W=6, L=3)):
        for prec in (32, 64):
            s = F.Solver(p, precision=prec, record_mm=True)
            s.iterate(3, 0.5); s.pass_(True, 0.5); s.pass_(False, 0.5); s.pass_(False, 0.5)
            s.lower_bound(); s.min_marginals(); s.finalize(); s.iterate(1, 0.5)
            try:
                s.round_primal(max_rounds=5)
            except F.FastdogError as e:
                assert e.code == 8
            s.close()
print("sanitize case ok")
