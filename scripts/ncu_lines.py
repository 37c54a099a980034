"""Summarise an ncu --page source --csv --print-source=cuda,sass dump per source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
key = sys.argv[2] if len(sys.argv) > 2 else "instr"
out = []
tot = tots = 0
fname = ""
idx = None
for row in rows:
    if not row:
        continue
    if row[0] in ("File Name", "File Path"):
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        idx = {h: i for i, h in enumerate(row)}
        continue
    if idx is None or row[0] == "":
        continue
    try:
        ie = int(row[idx["Instructions Executed"]])
        samp = int(row[idx["Warp Stall Sampling (All Samples)"]])
    except (ValueError, KeyError, IndexError):
        continue
    tot += ie
    tots += samp
    out.append((ie, samp, fname, row[0], row[1][:95]))
print("total warp instr", tot, "samples", tots)
k = 0 if key == "instr" else 1
for ie, samp, f, ln, src in sorted(out, key=lambda x: -x[k])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{ie:9d} {samp:6d} {f[:10]}:{ln}: {src}")
