#!/usr/bin/env python
"""Freeze the time-to-LB targets: for each bench workload, the
fp64 GPU bound after 1000 iterations (omega 0.5) from LB_0, recorded once per
(workload, seed) into bench_targets.json.  Run on a GPU box:
    python scripts/make_ttl_targets.py [workload ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2111_10270_b200 as F  # noqa: E402

names = sys.argv[1:] or ["mrf_potts", "gm_worms_like", "celltrack", "qap50"]
path = os.path.join(ROOT, "bench_targets.json")
data = json.load(open(path)) if os.path.exists(path) else {}
for name in names:
    p = bench._workload(name)
    s = F.Solver(p, precision=64, device=0)
    lb0 = s.lower_bound()
    s.iterate(1000, bench.OMEGA)
    data[p.name] = {"lb0_fp64": lb0, "lb_1000_fp64": s.lower_bound(), "iterations": 1000, "omega": bench.OMEGA,
                    "precision": 64}
    s.close()
    print(name, data[p.name], flush=True)
json.dump(data, open(path, "w"), indent=1, sort_keys=True)
