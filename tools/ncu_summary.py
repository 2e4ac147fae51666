"""Summarise ncu output into profiles/ (tracked):

    python tools/ncu_summary.py launches <launches.csv> <out.md>     # --metrics gpu__time_duration.sum list
    python tools/ncu_summary.py full <a.ncu-rep> [...] --out <out.md> [--traffic key=<rep> ...]

`full` reads each report with `ncu -i --page raw --csv` and writes per-kernel duration, DRAM
bytes, throughput and occupancy; `--traffic` also records DRAM bytes per launch into
profiles/traffic.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("dram__bytes.sum.per_second", "dram BW"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occ %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "inst"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9, "Tbyte/second": 1e12,
         "Tbyte/s": 1e12, "Gbyte/s": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def _num(v):
    return float(str(v).replace(",", ""))


def raw_rows(rep):
    if rep.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` exported on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, k in enumerate(hdr):
            if i < len(r):
                d[k] = (r[i], units[i])
        res.append(d)
    return res


def si(d, k):
    v, u = d[k]
    return _num(v) * SCALE.get(u, 1.0)


def full(reps, out, traffic):
    lines = ["# ncu --set full captures", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 (gpurun); "
             "times are cold-cache single launches under the profiler (not bench numbers).", ""]
    tr = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath))
    for rep in reps:
        for d in raw_rows(rep):
            name = d.get("Kernel Name", ("?", ""))[0]
            lines.append(f"## `{name[:150]}`")
            lines.append(f"report: `{os.path.basename(rep)}`")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for k, label in KEYS:
                if k in d:
                    v, u = d[k]
                    lines.append(f"| {label} (`{k}`) | {v} {u} |")
            if "dram__bytes_read.sum" in d:
                tot = si(d, "dram__bytes_read.sum") + si(d, "dram__bytes_write.sum")
                lines.append(f"| DRAM bytes per launch (rd+wr) | {tot:.4g} B |")
                for key, r2 in traffic:
                    if os.path.abspath(r2) == os.path.abspath(rep):
                        tr[key] = tot
            lines.append("")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        with open(tpath, "w") as f:
            json.dump(tr, f, indent=1, sort_keys=True)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    agg = collections.OrderedDict()
    n = 0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = _num(r[vi])
        except ValueError:
            continue
        unit = r[ui] if ui is not None else "nsecond"
        v *= SCALE.get(unit, 1e-9)
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        n += 1
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list: `{os.path.basename(path)}`", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold-cache per launch; "
             "shares, not absolute times, are comparable with the bench).", "",
             f"{n} launches, {tot * 1e3:.3f} ms total kernel time.", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{name}` | {c} | {t * 1e3:.3f} | {100 * t / tot:.1f}% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    a = sys.argv[1:]
    if a[0] == "launches":
        launches(a[1], a[2])
    else:
        reps, out, traffic = [], None, []
        i = 1
        while i < len(a):
            if a[i] == "--out":
                out = a[i + 1]
                i += 2
            elif a[i] == "--traffic":
                k, r = a[i + 1].split("=", 1)
                traffic.append((k, r))
                i += 2
            else:
                reps.append(a[i])
                i += 1
        full(reps, out, traffic)
