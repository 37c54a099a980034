"""Plan wall time per workload, host packer and GPU packer + compiler
(FDOG_GPU_PACK=1 FDOG_GPU_COMPILE=1), with the digests (identical); with
FDOG_PLAN_TRACE=1 the phases are printed to stderr."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_10270_b200 as F  # noqa: E402
import synth  # noqa: E402

for name in sys.argv[1:] or ["mrf_potts", "mrf_potts_cut", "celltrack", "qap50", "qap128"]:
    p = synth.WORKLOADS[name](0) if name in synth.WORKLOADS else synth.qap(0, 128)
    out = {}
    for mode in ("host", "gpu"):
        for k in ("FDOG_GPU_PACK", "FDOG_GPU_COMPILE"):
            os.environ.pop(k, None)
            if mode == "gpu":
                os.environ[k] = "1"
        t = time.perf_counter()
        pl = F.Plan(p, precision=32)
        out[mode] = (time.perf_counter() - t, pl.digest())
        pl.close()
    print(f"{name}: plan host {out['host'][0]:.2f} s, GPU pack + compile {out['gpu'][0]:.2f} s "
          f"({os.cpu_count()} host threads); digests equal: {out['host'][1] == out['gpu'][1]}", flush=True)
