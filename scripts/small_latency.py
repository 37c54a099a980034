"""Latency of tiny instances (BASELINE configs[0]): microseconds per iteration
of a warm iterate(n) loop, fused single-CTA path vs per-pass kernels (graphs)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_10270_b200 as F  # noqa: E402
import synth  # noqa: E402


def run(p, fused, precision, n=2000):
    os.environ["FDOG_FUSED"] = "1" if fused else "0"
    st = torch.cuda.Stream()
    s = F.Solver(p, precision=precision, stream=st.cuda_stream)
    s.iterate(10, 0.5)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    s.iterate(n, 0.5)
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n, s.lower_bound()


out = {}
for name, p in (("lap4_literal", synth.lap(synth.LAP4_LITERAL)), ("lap9_random", synth.lap_random(9, 5)),
                ("lap32_random", synth.lap_random(32, 1))):
    for prec in (32, 64):
        for fused in (False, True):
            us, lb = run(p, fused, prec)
            out[f"{name}/fp{prec}/{'fused' if fused else 'graph'}"] = {"us_per_iter": round(us, 3), "lb": lb}
print(json.dumps(out, indent=1))
