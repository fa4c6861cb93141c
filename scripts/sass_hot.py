"""Top stalled SASS instructions of an ncu report (source page, sass view).
  python scripts/sass_hot.py report.ncu-rep [N]"""
import csv, subprocess, sys, io
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_e = hdr.index("Instructions Executed")
tot = sum(int(r[i_s]) for r in data)
print("total samples", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
idx = sorted(range(len(data)), key=lambda i: -int(data[i][i_s]))[:n]
for i in sorted(idx):
    r = data[i]
    prev = data[i - 1][1].strip()[:60] if i else ""
    print(f"{i:5d} {int(r[i_s]):7d} {int(r[i_e]):10d}  {r[1].strip()[:70]:70s} | prev: {prev}")
