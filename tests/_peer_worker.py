"""Worker of tests/test_gpu_peer.py: one rank of a peer-exchange planning
job on cuda:0 (CUDA IPC works between processes on the same device; only one
of them ever runs a kernel, see the test's docstring).  Rendezvous through
files in a directory.

  python tests/_peer_worker.py DIR RANK WORLD MODE CYCLES
  MODE: solve (run CYCLES cycles of shard RANK of c2 K=3000 N=30 and write
        the folded results + per-candidate costs; on a failed exchange the
        per-candidate outputs) | idle (export, then sleep until DIR/stop
        appears; never runs a cycle; then dump what rank 0 stored into this
        rank's mailbox) | connect (only connect; prints CONNECTED or CONNECT_ERR)
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2603_20525_b200 import _abi, planner as PL  # noqa: E402
from parity_util import problem  # noqa: E402

d, rank, world, mode, cycles = Path(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
timeout_ms = int(sys.argv[6]) if len(sys.argv) > 6 else 30000
w, p, smp_full, terr, keep = problem("c2", 3000, 30)
k0, kc = PL.shard_range(3000, rank, world)
pl = PL.Planner(device=0, rank=rank, world_size=world, k_max=kc, n_steps_max=30,
                exchange=_abi.EXCHANGE_PEER, timeout_ms=timeout_ms)
pl.set_params(p)
pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
(d / f"h{rank}").write_bytes(pl.peer_export())
while not all((d / f"h{g}").exists() for g in range(world)):
    time.sleep(0.05)
time.sleep(0.2)
handles = [(d / f"h{g}").read_bytes() for g in range(world)]
if mode == "connect":  # only try to connect (the shared-GPU refusal)
    try:
        pl.peer_connect(handles)
        print("CONNECTED")
    except PL.ConfigError as e:
        print("CONNECT_ERR", e)
    (d / f"done{rank}").write_text("1")
    while not all((d / f"done{g}").exists() for g in range(world)):
        time.sleep(0.05)
    pl.close()
    sys.exit(0)
pl.peer_connect(handles)
(d / f"ready{rank}").write_text("1")
if mode == "idle":
    while not (d / "stop").exists():
        time.sleep(0.1)
    # what rank 0's kernel stored into this rank's mailbox for cycle 1
    rec, published = pl.peer_inspect(0, 1)
    np.savez(d / f"mailbox{rank}.npz", record=np.frombuffer(bytes(rec), dtype=np.uint8),
             published=published)
    pl.close()
    print("ok")
    sys.exit(0)
while not all((d / f"ready{g}").exists() for g in range(world)):
    time.sleep(0.05)
out = {}
try:
    for cyc in range(cycles):
        cfg = w.cfg.__class__(**{**w.cfg.__dict__, "n_samples": 3000, "n_steps": 30, "seed": 11 + cyc})
        smp, kk = PL.make_sampling(cfg, k0, kc)
        res, ctrl = pl.solve_raw(w.s0, smp)
        cost, flags, margin = pl.costs(kc)
        out[f"res{cyc}"] = np.frombuffer(bytes(res), dtype=np.uint8)
        out[f"cost{cyc}"] = cost
    np.savez(d / f"out{rank}.npz", **out)
    print("ok")
except RuntimeError as e:
    (d / f"err{rank}").write_text(str(e))
    # the kernel ran to its end: its per-candidate outputs are valid
    cost, flags, margin = pl.costs(kc)
    np.savez(d / f"outputs{rank}.npz", cost=cost, flags=flags, margin=margin)
    print("ERR", e)
pl.close()
