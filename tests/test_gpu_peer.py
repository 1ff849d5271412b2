"""The fused peer-memory record exchange (TMPC_EXCHANGE_PEER):
the rollout kernel's last block stores this GPU's reduction record into
every rank's mailbox over peer memory and waits for the others.

Only one kernel ever waits here: kernels that wait on one another must not
share a GPU (separate launches are not guaranteed to run at the same time;
on B200 two such processes raised Xid 109), and the test boxes have one GPU.
So the GPU side checks (a) a one-rank exchange (the kernel stores into its
own mailbox, publishes and finds the record) against the plain path over
several cycles (both mailbox buffers), and (b) two ranks where rank 1
connects but never runs a kernel: rank 0's kernel stores its record into
rank 1's mailbox through the CUDA IPC mapping, publishes, stops waiting after
timeout_ms and the call fails instead of hanging, and rank 1 finds rank 0's
record (equal to the host mirror of rank 0's outputs) and sequence number in
its mailbox.  The N-rank fold and the record plumbing are checked on the CPU
(tests/test_multi_rank.py, tests/test_bench_multirank.py)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2603_20525_b200 import _abi, planner as PL
from parity_util import problem

pytestmark = pytest.mark.gpu
WORKER = str(Path(__file__).resolve().parent / "_peer_worker.py")


def _env(allow):
    env = dict(os.environ)
    env.pop("TMPC_PEER_ALLOW_SHARED_GPU", None)
    if allow:
        env["TMPC_PEER_ALLOW_SHARED_GPU"] = "1"
    return env


def _strip_timing(b):
    r = _abi.tmpc_result.from_buffer_copy(bytes(b))
    r.kernel_ms = r.cycle_ms = 0.0
    return bytes(r)


def test_peer_exchange_one_rank_equals_plain():
    w, p, smp, terr, keep = problem("c2", 3000, 30)
    plain = PL.Planner(device=0, k_max=3000, n_steps_max=30)
    plain.set_params(p)
    plain.set_terrain_arrays(w.heights, w.sdist, w.grid)
    r0, c0 = plain.solve_raw(w.s0, smp)
    plain.close()
    pl = PL.Planner(device=0, k_max=3000, n_steps_max=30, exchange=_abi.EXCHANGE_PEER)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    pl.peer_connect([pl.peer_export()])
    for _ in range(3):  # both mailbox buffers
        r1, c1 = pl.solve_raw(w.s0, smp)
        assert _strip_timing(r1) == _strip_timing(r0)
        np.testing.assert_array_equal(c1, c0)
    assert pl.lib.tmpc_kernels_per_cycle(pl.ctx) == 2
    pl.close()


def test_peer_exchange_refuses_ranks_sharing_a_gpu(tmp_path):
    """Two ranks on one GPU: peer_connect fails with a ConfigError on both
    (their kernels would wait on one another) unless explicitly allowed."""
    procs = [subprocess.Popen([sys.executable, WORKER, str(tmp_path), str(r), "2", "connect", "0"],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                              env=_env(allow=False)) for r in range(2)]
    for pr in procs:
        so, se = pr.communicate(timeout=300)
        assert pr.returncode == 0, se[-3000:]
        assert "CONNECT_ERR" in so and "share GPU" in so, so


def test_peer_exchange_missing_rank_times_out(tmp_path):
    """Rank 1 connects but never runs a cycle: rank 0's kernel stores its
    record into rank 1's mailbox, stops waiting after timeout_ms and the call
    fails (no hang); rank 1's mailbox then holds rank 0's record of sequence
    number 1, equal to the host mirror of rank 0's per-candidate outputs."""
    # two ranks on the test box's one GPU, allowed here: rank 1 never launches,
    # so only rank 0's kernel waits
    idle = subprocess.Popen([sys.executable, WORKER, str(tmp_path), "1", "2", "idle", "0"],
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                            env=_env(allow=True))
    r0 = subprocess.run([sys.executable, WORKER, str(tmp_path), "0", "2", "solve", "1", "2000"],
                        capture_output=True, text=True, timeout=300, env=_env(allow=True))
    (tmp_path / "stop").write_text("1")
    so, se = idle.communicate(timeout=120)
    assert r0.returncode == 0, r0.stderr[-3000:]
    assert "ERR" in r0.stdout and "did not arrive" in r0.stdout, r0.stdout
    assert idle.returncode == 0 and "ok" in so, se[-3000:] + so
    got = np.load(tmp_path / "mailbox1.npz")
    out0 = np.load(tmp_path / "outputs0.npz")
    assert int(got["published"]) == 1
    rec = _abi.tmpc_rank_record.from_buffer_copy(got["record"].tobytes())
    want = PL.make_record(out0["cost"], out0["flags"], out0["margin"], 0)
    assert (rec.k_begin, rec.k_count) == (0, 1500)
    for f in ("key_lo", "key_hi", "min_cost_bits", "n_feasible", "n_diverged", "n_goal",
              "n_finite", "best_cost", "best_flags", "best_margin"):
        assert getattr(rec, f) == getattr(want, f), f
    assert list(rec.cost_limb) == list(want.cost_limb)
