import os, sys
os.environ["FDOG_TRACE"] = "1"; os.environ["FDOG_GRAPHS"] = "0"
sys.path.insert(0, os.getcwd())
import numpy as np
import synth, paper_2111_10270_b200 as F
for name, mk in (("celltrack", lambda: synth.celltrack(0)), ("qap50", lambda: synth.qap(0, 50))):
    p = mk()
    for cb in ("1", "2"):
        os.environ["FDOG_CLAIM"] = cb
        s = F.Solver(p, precision=32)
        s.iterate(3, 0.5); s.pass_(True, 0.5)
        tr = s.debug_trace().astype(np.int64)
        t0 = tr[:, 0].min()
        st, en, nt, sm = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, tr[:, 2], tr[:, 3]
        o = np.argsort(-en)[:6]
        print(name, "claim", cb, "span %.1f p90 %.1f" % (en.max(), np.percentile(en, 90)),
              [(int(w), round(float(en[w]), 1), int(nt[w]), int(sm[w]), int((sm == sm[w]).sum())) for w in o])
        # per SM: warps and total tiles of the straggler's SM vs median
        s.close()
