"""Pivot an `ncu --csv --metrics ...` log (one row per kernel x metric) into a
per-launch table.  Usage: python profiles/ncu_table.py LOG [max_rows]"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
rows = rows[next(i for i, r in enumerate(rows) if r[0] == "ID"):]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki]), OrderedDict())[r[mi]] = r[vi]
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 60
for (i, k), v in list(d.items())[:lim]:
    name = k.split("(")[0].replace("void ", "")[:44]
    print(f"{i:>4} {name:44s} " + " ".join(f"{m.split('__')[1][:18]}={v[m]}" for m in v))
