"""Top stalled SASS instructions of an ncu report (--import-source on),
appended to a profiles/ summary (dev tool; reads a local .ncu-rep)."""
import csv
import subprocess
import sys
from pathlib import Path

rep, out = sys.argv[1], Path(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, data = rows[1], rows[2:]
isrc = hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
inot = hdr.index("Warp Stall Sampling (Not-issued Samples)")
iex = hdr.index("Instructions Executed")
tot = sum(int(r[iall]) for r in data) or 1
lines = ["", f"top {n} SASS instructions by not-issued stall samples ({tot} samples):"]
for i in sorted(range(len(data)), key=lambda i: -int(data[i][inot]))[:n]:
    r = data[i]
    lines.append(f"  #{i:5d} {100 * int(r[inot]) / tot:5.1f}%  exec {int(r[iex]):>9d}  {r[isrc].strip()[:70]}")
with out.open("a") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
