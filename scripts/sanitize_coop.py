"""compute-sanitizer target: a small knapsack-style instance (cooperative tiles), fp32 and fp64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_10270_b200 as F  # noqa: E402
import synth  # noqa: E402

for prec in (64, 32):
    p = synth.gap(1, jobs=40, agents=5)
    g = F.Solver(p, precision=prec, record_mm=True)
    g.iterate(2, 0.5)
    print(prec, g.lower_bound())
