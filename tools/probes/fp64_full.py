"""fp64 certification mode at full c4 / c5 size against oracle/_ref (dev probe)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
from paper_2603_20525_b200 import _abi
import test_gpu_parity as T
from parity_util import best_oracle, check_parity
orc = best_oracle()
for name in sys.argv[1:]:
    w, p, smp, terr, keep = T._full(name)
    res, ctrl, cost, flags, margin = T._device(w, p, smp, _abi.PRECISION_FP64)
    st = check_parity(orc, w, p, smp, terr, w.s0, cost, flags, margin, res.best_index, threads=16,
                      label=f"{name} fp64", spread_all=False)
    print("RESULT", name, st, flush=True)
