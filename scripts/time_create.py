import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2111_10270_b200 as F
p = synth.gm_worms_like(0)
t = time.perf_counter(); plan = F.Plan(p); print("plan %.1f ms" % ((time.perf_counter() - t) * 1e3))
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    s = F.Solver(plan=plan, precision=32)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s.iterate(50, 0.5); s.lower_bound(); t2 = time.perf_counter()
    lam = s.lam(); t3 = time.perf_counter()
    print("create %.1f ms, 50 iters+lb %.1f ms, get_lambda %.1f ms, device MB %.1f" % ((t1 - t) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, s.stats()["device_bytes"] / 1e6))
    s.close()
