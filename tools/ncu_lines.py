"""Aggregate an ncu source page (--print-source=cuda,sass --csv) by CUDA source line.

usage: ncu -i rep --page source --csv --print-source=cuda,sass | python tools/ncu_lines.py [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
n_top = int(sys.argv[1]) if len(sys.argv) > 1 else 40
agg = defaultdict(lambda: [0.0, 0.0, ""])
stall_cols = None
stall_agg = defaultdict(float)
cur_file = "?"
h = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        wi = h.index("Warp Stall Sampling (All Samples)")
        ii = h.index("Instructions Executed")
        stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if h is None or len(r) <= wi or not r[0].isdigit():
        continue
    key = (cur_file, int(r[0]))
    try:
        agg[key][0] += float(r[wi] or 0)
        agg[key][1] += float(r[ii] or 0)
    except ValueError:
        pass
    agg[key][2] = r[1].strip()[:90]
    for i, c in stall_cols:
        try:
            stall_agg[c] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot:.0f}")
for (f, ln), (w, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n_top]:
    print(f"{f:18s}{ln:5d} {w:7.0f} {100*w/tot:5.1f}% inst={ins:9.0f}  {src}")
st = sum(stall_agg.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]}={100*v/st:.1f}%" for k, v in sorted(stall_agg.items(), key=lambda kv: -kv[1])[:8]))
