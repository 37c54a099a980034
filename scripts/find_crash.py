"""Run the random tiny ILPs one by one (for compute-sanitizer): prints the seed before each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2111_10270_b200 as F
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 200):
    p = synth.random_ilp(seed, n=10, m=7, kmax=7, coef=3)
    print("seed", seed, flush=True)
    g = F.Solver(p, precision=64, record_mm=True)
    st = g.stats()
    print(" tiles", st["tiles"], "staged", st["staged_tiles"], "rc", st["sweep_recompute"], "stream", st["sweep_streaming"],
          "fused", st["fused_small"], "maxw", st["max_width"], flush=True)
    for t in range(2):
        g.pass_(t % 2 == 0, 0.5)
        g.lam(); g.deferred(); g.min_marginals(); g.lower_bound()
    g.close()
print("ok")
