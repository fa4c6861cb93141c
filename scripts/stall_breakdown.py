"""Stall-reason breakdown of an ncu report's SASS lines in [lo, hi) (sass_hot.py indices).
  python scripts/stall_breakdown.py report.ncu-rep lo hi"""
import csv, subprocess, io, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); hdr = rows[1]; data = rows[2:]
lo, hi = int(sys.argv[2]), int(sys.argv[3])
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: 0 for c in cols}
for i in range(lo, hi):
    for c in cols:
        v = data[i][hdr.index(c)]
        agg[c] += int(v) if v not in ("", "-") else 0
for c, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"{c:28s} {v}")
top = sorted(range(lo, hi), key=lambda i: -int(data[i][hdr.index("Warp Stall Sampling (All Samples)")]))[:12]
for i in sorted(top):
    print(i, data[i][hdr.index("Warp Stall Sampling (All Samples)")], data[i][1].strip()[:80])
