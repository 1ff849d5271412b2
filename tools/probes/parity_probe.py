"""Full-size fp32 parity of one (config, model, scheme) under the north-star
rule (tests/parity_util.check_parity), printed instead of asserted (dev
probe, to try a case before it becomes a test).

  python tools/probes/parity_probe.py c4:1:1 c5:0:1 ...   (config:model:scheme[:fp64])
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2603_20525_b200 import _abi  # noqa: E402
import test_gpu_parity as T  # noqa: E402
from parity_util import best_oracle, check_parity  # noqa: E402

orc = best_oracle()
for spec in sys.argv[1:]:
    parts = spec.split(":")
    name, model, scheme = parts[:3]
    prec = _abi.PRECISION_FP64 if len(parts) > 3 and parts[3] == "fp64" else _abi.PRECISION_FP32
    w, p, smp, terr, keep = T._full(name)
    p.model, p.scheme = int(model), int(scheme)
    res, ctrl, cost, flags, margin = T._device(w, p, smp, prec)
    try:
        st = check_parity(orc, w, p, smp, terr, w.s0, cost, flags, margin, res.best_index,
                          threads=16, label=f"{spec}", spread_all=False)
        print("PASS", spec, st, flush=True)
    except AssertionError as e:
        print("FAIL", spec, str(e)[:1500], flush=True)
