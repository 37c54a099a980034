"""Where the e2e time goes (GM, fp32): create from plan, K x (iterate(1) + lower_bound), get_lambda."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2111_10270_b200 as F
p = synth.gm_worms_like(0)
plan = F.Plan(p, precision=32)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = F.Solver(plan=plan, precision=32, stream=stream.cuda_stream)
    t1 = time.perf_counter()
    for _ in range(50):
        s.iterate(1, 0.5)
        s.lower_bound()
    t2 = time.perf_counter()
    lam = s.lam()
    t3 = time.perf_counter()
    s.close()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms | 50 x (iterate+lb) {1e3*(t2-t1):.2f} ms ({1e6*(t2-t1)/50:.1f} us/step) | get_lambda {1e3*(t3-t2):.2f} ms | close {1e3*(t4-t3):.2f} ms")
