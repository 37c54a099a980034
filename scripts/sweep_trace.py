"""Per-warp timeline of one sweep (FDOG_TRACE=1): when warps start / finish, per SM."""
import os, sys
os.environ["FDOG_TRACE"] = "1"
os.environ["FDOG_GRAPHS"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth, paper_2111_10270_b200 as F
for name in sys.argv[1:] or ["celltrack"]:
    p = {"gm_worms_like": lambda: synth.gm_worms_like(0), "celltrack": lambda: synth.celltrack(0),
         "qap50": lambda: synth.qap(0, 50), "mrf_potts": lambda: synth.mrf_potts(0)}[name]()
    s = F.Solver(p, precision=32)
    s.iterate(3, 0.5)
    s.pass_(True, 0.5)
    tr = s.debug_trace().astype(np.int64)
    t0 = tr[:, 0].min()
    st, en, nt, sm = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, tr[:, 2], tr[:, 3]
    span = en.max()
    sm_end = np.array([en[sm == q].max() for q in np.unique(sm)])
    sm_start = np.array([st[sm == q].min() for q in np.unique(sm)])
    print(f"{name}: warps {len(tr)}, span {span:.1f} us; warp start: max {st.max():.2f} us; "
          f"warp end: min {en.min():.1f} p10 {np.percentile(en,10):.1f} p50 {np.percentile(en,50):.1f} p90 {np.percentile(en,90):.1f} max {en.max():.1f}; "
          f"SM end: min {sm_end.min():.1f} p50 {np.median(sm_end):.1f}; tiles/warp min {nt.min()} max {nt.max()} mean {nt.mean():.1f}")
    busy = (en - st).sum() / (len(tr) * span)
    print(f"   warp-busy fraction of span {busy:.2f}; SMs {len(sm_end)}")
    s.close()
