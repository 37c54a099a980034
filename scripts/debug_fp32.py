import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
import paper_2111_10270_b200 as F
p = synth.gm_worms_like(5, n_src=120, k_cand=8, knn=10)
o = oracle.Oracle(p)
for graphs in ("0", "1"):
    os.environ["FDOG_GRAPHS"] = graphs
    o = oracle.Oracle(p)
    g = F.Solver(p, precision=32)
    print("graphs", graphs, g.stats()["tiles"], g.stats()["staged_tiles"], g.stats()["sweep_smem_per_warp"])
    for t in range(12):
        if graphs == "0":
            g.pass_(t % 2 == 0, 0.5); o.pass_(t % 2 == 0, 0.5)
        else:
            if t % 2: continue
            g.iterate(1, 0.5); o.iterate(1, 0.5)
        dl = np.max(np.abs(g.lam() - o.lam()))
        print(t, "lb", g.lower_bound(), o.lower_bound(), "max dlam", dl, "argmax", int(np.argmax(np.abs(g.lam() - o.lam()))))
    p64 = F.Solver(p, precision=64)
    o = oracle.Oracle(p)
    p64.iterate(5, 0.5); o.iterate(5, 0.5)
    print("fp64 after 5:", p64.lower_bound(), o.lower_bound())
