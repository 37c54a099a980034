"""A/B: iteration time of a workload with two builds of the package (same box)."""
import os, sys
pkg, name = sys.argv[1], sys.argv[2]
sys.path.insert(0, pkg)
import torch
import synth
import paper_2111_10270_b200 as F
assert F.__file__.startswith(os.path.abspath(pkg)), F.__file__
p = {"mrf_potts": lambda: synth.mrf_potts(0), "qap50": lambda: synth.qap(0, 50),
     "celltrack": lambda: synth.celltrack(0), "gm_worms_like": lambda: synth.gm_worms_like(0)}[name]()
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
s = F.Solver(p, precision=32, stream=st.cuda_stream)
s.iterate(5, 0.5); torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
res = []
for rep in range(3):
    a.record(st); s.iterate(20, 0.5); b.record(st); torch.cuda.synchronize()
    res.append(a.elapsed_time(b) / 20 * 1e3)
print(f"{os.path.basename(pkg)} {name}: us/iteration {min(res):.1f} (reps {', '.join(f'{x:.1f}' for x in res)})")
