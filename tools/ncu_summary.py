"""Summarise an ncu --csv launch list: per kernel name, launches and metric means."""
import csv
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = defaultdict(lambda: defaultdict(list))
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        per[name][r[mi]].append(float(r[vi].replace(",", "")))
    print(f)
    for name, mets in per.items():
        parts = [f"{m}={sum(v)/len(v):,.1f}" for m, v in sorted(mets.items())]
        print(f"  {name[:60]:60s} n={len(next(iter(mets.values())))} " + " ".join(parts))
