"""Summarise an ncu --metrics CSV (one row per kernel launch x metric) into per-kernel medians."""
import collections
import csv
import statistics
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault(r[iid], {"k": r[ik].split("(")[0]})[r[im]] = float(r[iv].replace(",", ""))
groups = collections.OrderedDict()
for d in per.values():
    groups.setdefault(d["k"], []).append(d)
for k, ds in groups.items():
    keys = [m for m in ds[0] if m != "k"]
    print(k, len(ds), {m.replace("sm__", "").replace("smsp__", "")[:28]: round(statistics.median(d[m] for d in ds), 3)
                       for m in keys})
