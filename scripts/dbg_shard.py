"""Debug: sharded GM solve in external-exchange mode, printing solver stats."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth, paper_2111_10270_b200 as F
p = synth.gm_worms_like(12, n_src=60, k_cand=6, knn=6)
world = 2
ranks = [F.Solver(p, precision=64, rank=r, world=world) for r in range(world)]
for g in ranks:
    st = g.stats()
    print({k: st[k] for k in ("tiles", "staged_tiles", "sweep_grid", "sweep_block", "sweep_smem_per_warp",
                              "sweep_streaming", "sweep_recompute", "fused_small")}, flush=True)
for t in range(6):
    fwd = t % 2 == 0
    for g in ranks:
        g.pass_begin(fwd, 0.5)
    x = sum(g.exchange_read() for g in ranks)
    for g in ranks:
        g.exchange_write(x)
    for i, g in enumerate(ranks):
        print("pass", t, "rank", i, flush=True)
        g.pass_end(fwd, 0.5)
print("ok")
