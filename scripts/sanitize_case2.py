"""compute-sanitizer case for the round's later kernels: non-deferred (seq) passes, the
chunked sweep (long rows), the GPU BDD compiler, and the root/join-folded tiles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
import paper_2111_10270_b200 as F
os.environ["FDOG_GPU_COMPILE"] = "1"
rng = np.random.default_rng(0)
rows = [(np.sort(rng.choice(1500, size=900, replace=False)), np.ones(900), synth.LE, 1) for _ in range(3)]
rows += [(np.array([q, q + 1]), np.ones(2), synth.LE, 1) for q in range(0, 1499, 2)]
long_rows = synth.from_rows(1500, rng.uniform(-1, 1, 1500), rows, "long")
for p in (synth.gm_worms_like(3, n_src=40, k_cand=4, knn=4), synth.mrf_potts(3, H=5, W=6, L=3),
          synth.random_ilp(7, n=40, m=60, kmax=12, coef=5), long_rows, synth.thin_hop(3, k=700)):
    for prec in (32, 64):
        s = F.Solver(p, precision=prec, record_mm=True)
        s.iterate(2, 0.5); s.pass_(True, 0.5); s.pass_(False, 0.5)
        s.lower_bound(); s.min_marginals(); s.finalize()
        s.iterate_seq(2, 0.5); s.pass_seq(True, 0.5)
        s.lower_bound(); s.lam(); s.min_marginals()
        s.close()
print("sanitize case 2 ok")
