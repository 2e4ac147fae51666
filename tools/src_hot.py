"""Summarise an ncu source-page CSV export (--page source --csv --print-source cuda,sass):
stall samples per CUDA source line (top N) and per stall reason.
    python tools/src_hot.py gpurun_out/x.source.csv [N]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
h = rows[hi[0]]
idx = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
per_line = defaultdict(lambda: [0, 0, defaultdict(float), ""])
tot = 0
reasons = defaultdict(float)
for r in rows[hi[0] + 1:]:
    if len(r) < len(h) or not r[0].strip():
        continue
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        ins = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    e = per_line[r[0]]
    e[0] += s
    e[1] += ins
    e[3] = r[1][:100].strip()
    tot += s
    for n in stalls:
        v = float(r[idx[n]] or 0)
        e[2][n] += v
        reasons[n] += v
print("total samples", tot)
print("reasons:", ", ".join(f"{k[6:]} {v / max(tot, 1):.1%}" for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:8]))
for line, (s, ins, st, src) in sorted(per_line.items(), key=lambda x: -x[1][0])[:top]:
    best = sorted(st.items(), key=lambda x: -x[1])[:2]
    print(f"{s:6d} {s / max(tot, 1):6.1%} ins {ins:8d}  L{line:>4} {src[:70]:70s} " +
          " ".join(f"{k[6:]}={v:.0f}" for k, v in best))
