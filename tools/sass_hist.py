"""Opcode histogram of the per-substep loop body of a rollout kernel (SASS).

usage: python tools/sass_hist.py [kernel-substring]  (default rollout_kernel_f32ILi1)
Finds the largest backward branch (the substep loop), then the body that the
q != 0 path executes (from the uniform branch that skips the ZOH-boundary
block to the back-edge) and prints the opcode counts."""
import collections
import os
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(os.environ.get("TMPC_B200_LIB", Path(__file__).resolve().parents[1] / "paper_2603_20525_b200" / "libtmpc_b200.so"))
pat = sys.argv[1] if len(sys.argv) > 1 else "rollout_kernel_f32ILi1"
sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs if f.split("\n", 1)[0].find(pat) >= 0)
ins = []
for line in body.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for a, t in ins:
    m = re.search(r"BRA\S*\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        loops.append((a - int(m.group(1), 16), int(m.group(1), 16), a))
span, lo, hi = max(loops)
# the first uniform forward branch at the loop head skips the ZOH block
start = lo
for a, t in ins:
    if lo <= a <= lo + 0x40 and "BRA.U" in t:
        start = int(re.search(r"0x([0-9a-f]+)", t.split("BRA")[1]).group(1), 16)
        break
c = collections.Counter()
n = 0
for a, t in ins:
    if start <= a <= hi:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        c[op.split(".")[0]] += 1
        n += 1
print(f"{pat}: loop {lo:#x}-{hi:#x}, substep path {start:#x}-{hi:#x}: {n} instructions")
for op, k in c.most_common(30):
    print(f"{k:5d} {op}")
