"""Summarise a round's ncu captures into profiles/ (committed evidence).

usage: python scripts/summarize_ncu.py TAG [bench.json]
  reads gpurun_out/launches_TAG.csv (launch list, gpu__time_duration) and
  gpurun_out/prof_TAG.ncu-rep (--set full capture); writes
  profiles/TAG_launches.csv and profiles/TAG_ncu_summary.md.  (bench.py
  measures roofline.traffic itself, with an ncu subprocess of the same run.)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles")
os.makedirs(out, exist_ok=True)
lines = []

# launch list
lp = os.path.join(root, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(lp):
    txt = "".join(l for l in open(lp) if not l.startswith("=="))
    rows = list(csv.DictReader(io.StringIO(txt)))
    with open(os.path.join(out, f"{tag}_launches.csv"), "w") as f:
        f.write("id,kernel,grid,block,gpu__time_duration_ns\n")
        for r in rows:
            f.write(f"{r['ID']},\"{r['Kernel Name'][:80]}\",\"{r['Grid Size']}\",\"{r['Block Size']}\",{r['Metric Value']}\n")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    lines.append(f"## Launch list ({lp.split('/')[-1]}; ncu gpu__time_duration.sum, --clock-control none, cold-cache serialised)\n")
    lines.append("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {ns/1e3:.1f} | {ns/n/1e3:.2f} | {ns/tot:.3f} |")
    lines.append("")

# full captures: prof_TAG.ncu-rep and prof_TAG_<workload>_<kernel>.ncu-rep
import glob  # noqa: E402
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for rp in sorted(glob.glob(os.path.join(root, "gpurun_out", f"prof_{tag}.ncu-rep")) +
                 glob.glob(os.path.join(root, "gpurun_out", f"prof_{tag}_*.ncu-rep")) +
                 glob.glob(os.path.join(root, "gpurun_out", f"prof_{tag}_*.raw.csv"))):
    if rp.endswith(".raw.csv"):  # exported on the box (scripts/gpu_ncu.sh)
        raw = open(rp).read()
    else:
        raw = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) < 3:
        continue
    hdr, units = rr[0], rr[1]
    lines.append(f"## ncu --set full ({rp.split('/')[-1]})\n")
    for row in rr[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        lines.append(f"`{name}`\n")
        lines.append("| metric | value |\n|---|---|")
        for w in want:
            if w in d:
                lines.append(f"| {w} | {d[w]} {u.get(w, '')} |")
        ld_r = d.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "")
        st_r = d.get("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "")
        try:
            lines.append(f"| sectors per global load request | "
                         f"{float(d['l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum'].replace(',', '')) / float(ld_r.replace(',', '')):.2f} |")
            lines.append(f"| sectors per global store request | "
                         f"{float(d['l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum'].replace(',', '')) / float(st_r.replace(',', '')):.2f} |")
        except (KeyError, ValueError, ZeroDivisionError):
            pass
        st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("per_issue_active.ratio") and v not in ("", "n/a")}
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        lines.append("\nstalls (cycles per issued instruction): " + ", ".join(f"{k} {v:.2f}" for k, v in top) + "\n")

if len(sys.argv) > 2 and os.path.exists(sys.argv[2]):
    b = json.load(open(sys.argv[2]))
    lines.insert(0, f"Bench line of the same round ({sys.argv[2].split('/')[-1]}): value {b['value']:.4g} {b['unit']}, "
                    f"{b['ms_per_step']*1e3:.1f} us/step, roofline frac {b['roofline']['frac']:.3f} "
                    f"({b['roofline']['achieved']:.0f} of {b['roofline']['peak']} GB/s {b['roofline']['peak_kind']}), "
                    f"kernel shares {json.dumps({k: round(v, 3) for k, v in b['kernel_share'].items()})}\n")
lines.insert(0, f"# ncu summary, {tag}\n")
with open(os.path.join(out, f"{tag}_ncu_summary.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
