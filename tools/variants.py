"""Build a kernel variant library (dev tool): variants/NAME/libtmpc_b200.so
compiled with extra preprocessor flags, for tools/ab.py.

  python tools/variants.py NAME "-DTMPC_X=1 -DTMPC_Y=0"
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
name, flags = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
d = ROOT / "variants" / name
d.mkdir(parents=True, exist_ok=True)
(d / "flags.txt").write_text(flags + "\n")
subprocess.run(["make", "-s", "-C", str(ROOT / "paper_2603_20525_b200" / "csrc"),
                f"OUT={d / 'libtmpc_b200.so'}", f"PTXLOG={d / 'ptxas.log'}", f"EXTRA={flags}"],
               check=True)
