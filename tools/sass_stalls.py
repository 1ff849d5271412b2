"""Static schedule of the per-substep loop body of a rollout kernel (dev tool).

usage: python tools/sass_stalls.py [kernel-substring] [--dump]
Decodes the Volta+ control bits of each SASS instruction in the substep path
(same region as tools/sass_hist.py): stall cycles (bits 105-108), yield (109),
write / read scoreboard (110-115) and wait mask (116-121).  The sum of the
stall fields is the number of cycles one warp alone needs per substep before
any scoreboard (variable-latency: LDG/TLD, MUFU, SHFL, LDC) wait -- a CPU-side
lower bound for the lone-warp chain, to compare schedules without a GPU."""
import collections
import os
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(os.environ.get("TMPC_B200_LIB", Path(__file__).resolve().parents[1] / "paper_2603_20525_b200" / "libtmpc_b200.so"))
args = [a for a in sys.argv[1:] if not a.startswith("--")]
pat = args[0] if args else "rollout_kernel_f32ILi1ELi1ELi0"
sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs if f.split("\n", 1)[0].find(pat) >= 0)
ins = []
lines = body.splitlines()
for i, line in enumerate(lines):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* 0x([0-9a-f]{16}) \*/", line)
    if m:
        hi = int(re.search(r"0x([0-9a-f]{16})", lines[i + 1]).group(1), 16)
        ins.append((int(m.group(1), 16), m.group(2).strip(), hi))
loops = []
for a, t, _ in ins:
    m = re.search(r"BRA\S*\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        loops.append((a - int(m.group(1), 16), int(m.group(1), 16), a))
span, lo, hi_addr = max(loops)
start = lo
for a, t, _ in ins:
    if lo <= a <= lo + 0x40 and "BRA.U" in t:
        start = int(re.search(r"0x([0-9a-f]+)", t.split("BRA")[1]).group(1), 16)
        break
n = stall_sum = waits = 0
by_stall = collections.Counter()
op_stall = collections.Counter()
for a, t, h in ins:
    if not (start <= a <= hi_addr):
        continue
    stall = (h >> 41) & 0xF
    wmask = (h >> 52) & 0x3F
    n += 1
    stall_sum += stall
    by_stall[stall] += 1
    op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
    op_stall[op] += stall
    waits += wmask != 0
    if "--dump" in sys.argv:
        print(f"{a:06x} st{stall:2d} w{wmask:02x} {t}")
print(f"{pat}: {n} instructions, stall-cycle sum {stall_sum} (lone-warp lower bound per substep), "
      f"{waits} scoreboard waits")
print("stall histogram:", dict(sorted(by_stall.items())))
print("stall cycles by opcode:", op_stall.most_common(12))
