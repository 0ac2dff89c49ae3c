"""Summarise an ncu launch list (gpu__time_duration + dram bytes, --csv) by
kernel in launch order, collapsing runs: python scripts/launch_summary.py file.csv [--md]"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
md = "--md" in sys.argv
rows = list(csv.reader(open(path)))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr, start = r, i
        break
ki, mi, vi, ui, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
recs = defaultdict(dict)
names = {}
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    sc = {"ns": 1e-3, "us": 1, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
    recs[int(r[idi])][r[mi]] = v * sc
    names[int(r[idi])] = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("lb::", "")[:60]
ids = sorted(recs)
tot = sum(recs[i]["gpu__time_duration.sum"] for i in ids)
out = []
prev, acc = None, [0, 0.0, 0.0, 0.0]
def flush():
    if prev:
        out.append((prev, *acc))
for i in ids:
    n, m = names[i], recs[i]
    if n != prev:
        flush()
        prev, acc = n, [0, 0.0, 0.0, 0.0]
    acc[0] += 1
    acc[1] += m["gpu__time_duration.sum"]
    acc[2] += m.get("dram__bytes_read.sum", 0)
    acc[3] += m.get("dram__bytes_write.sum", 0)
flush()
if md:
    print(f"{len(ids)} launches, {tot:.1f} us in total (ncu: serialised, cold caches; compare shares)\n")
    print("| kernel | launches | us | share | DRAM read MB | DRAM write MB |\n|---|---|---|---|---|---|")
    for n, c, t, rd, wr in out:
        print(f"| `{n}` | {c} | {t:.1f} | {100 * t / tot:.1f}% | {rd / 1e6:.1f} | {wr / 1e6:.1f} |")
else:
    print("launches", len(ids), "total us", tot)
    for n, c, t, rd, wr in out:
        print(f"{n:60s} x{c:3d} {t:9.1f} us {100 * t / tot:5.1f}%  rd {rd / 1e6:8.1f} MB wr {wr / 1e6:8.1f} MB")
