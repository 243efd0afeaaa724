"""Per-source-line stall samples / executed instructions from an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass,cuda > X.csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
S = hdr.index("Warp Stall Sampling (All Samples)")
E = hdr.index("Instructions Executed")
W = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
lines = [r for r in rows[3:] if len(r) == len(hdr) and r[0] not in ("", "Line No")]
tot = sum(int(r[S]) for r in lines if r[S].isdigit())
tot_e = sum(int(r[E]) for r in lines if r[E].isdigit())
print(f"total samples {tot}, instructions {tot_e}")
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
for r in lines:
    s = int(r[S]) if r[S].isdigit() else 0
    e = int(r[E]) if r[E].isdigit() else 0
    w = int(r[W]) if W is not None and r[W].isdigit() else 0
    if s > thr * tot or e > thr * tot_e:
        print(f"{r[0]:>5s} {100 * s / tot:5.1f}% samp {100 * e / tot_e:5.1f}% inst wf {w:8d}  {r[1].strip()[:80]}")
