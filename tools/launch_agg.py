"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) of `prof_op.py <cfg> 9 2`
(two eager cycles): per kernel and grid of the SECOND cycle, count, total and mean microseconds.
    python tools/launch_agg.py gpurun_out/launches_c4.csv [top]"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[0]
ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
recs = [(r[ki], r[gi], float(r[vi].replace(",", "")) / 1000.0) for r in rows[1:]]
cyc = recs[len(recs) // 2:]
agg = defaultdict(lambda: [0, 0.0])
for k, g, t in cyc:
    key = (re.sub(r"\(.*", "", k)[:72], g)
    agg[key][0] += 1
    agg[key][1] += t
tot = sum(t for _, _, t in cyc)
print("launches", len(cyc), "sum us", round(tot, 1))
for (k, g), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{t:9.1f} us {t / tot:6.1%} {c:4d}x {t / c:8.2f}  {g:16s} {k}")
