"""Host plan wall time per workload (FDOG_PLAN_TRACE=1 prints the phases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2111_10270_b200 as F
for name in sys.argv[1:] or ["gm_worms_like", "mrf_potts", "celltrack", "qap50", "qap128"]:
    p = {"gm_worms_like": lambda: synth.gm_worms_like(0), "mrf_potts": lambda: synth.mrf_potts(0),
         "celltrack": lambda: synth.celltrack(0), "qap50": lambda: synth.qap(0, 50),
         "qap128": lambda: synth.qap(0, 128)}[name]()
    t = time.perf_counter()
    pl = F.Plan(p, precision=32)
    print(f"{name}: plan {time.perf_counter() - t:.2f} s on {os.cpu_count()} host threads", flush=True)
    pl.close()
