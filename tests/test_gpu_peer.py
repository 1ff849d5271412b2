"""The fused peer-memory record exchange (TMPC_EXCHANGE_PEER):
the rollout kernel's last block stores this GPU's reduction record into
every rank's mailbox over peer memory and waits for the others -- checked
with several processes on one GPU (CUDA IPC works between processes on the
same device): the folded result of every rank equals the one-process solve
bit for bit over several cycles (both mailbox buffers), per-candidate
outputs reassemble, and a rank that never runs its cycle makes the others
fail after their timeout instead of hanging."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2603_20525_b200 import _abi, planner as PL
from parity_util import problem

pytestmark = pytest.mark.gpu
WORKER = str(Path(__file__).resolve().parent / "_peer_worker.py")


def _one_process(cycles):
    w, p, smp, terr, keep = problem("c2", 3000, 30)
    pl = PL.Planner(device=0, k_max=3000, n_steps_max=30)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    out = []
    for cyc in range(cycles):
        cfg = w.cfg.__class__(**{**w.cfg.__dict__, "n_samples": 3000, "n_steps": 30,
                                 "seed": 11 + cyc})
        smp, kk = PL.make_sampling(cfg)
        res, ctrl = pl.solve_raw(w.s0, smp)
        out.append((bytes(res), pl.costs(3000)[0].copy()))
    pl.close()
    return out


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


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_processes_on_one_gpu(tmp_path, world):
    cycles = 3
    procs = [subprocess.Popen([sys.executable, WORKER, str(tmp_path), str(r), str(world), "solve",
                               str(cycles)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(world)]
    outs = [pr.communicate(timeout=600) for pr in procs]
    for pr, (so, se) in zip(procs, outs):
        assert pr.returncode == 0 and "ok" in so, se[-3000:] + so
    ref = _one_process(cycles)
    for cyc in range(cycles):
        costs = []
        for r in range(world):
            z = np.load(tmp_path / f"out{r}.npz")
            assert _strip_timing(z[f"res{cyc}"]) == _strip_timing(ref[cyc][0]), (r, cyc)
            costs.append(z[f"cost{cyc}"])
        np.testing.assert_array_equal(np.concatenate(costs), ref[cyc][1])


def test_peer_exchange_missing_rank_times_out(tmp_path):
    """Rank 1 connects but never runs a cycle: rank 0's kernel stops waiting
    after timeout_ms and the call fails (no hang)."""
    idle = subprocess.Popen([sys.executable, WORKER, str(tmp_path), "1", "2", "idle", "0"],
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    r0 = subprocess.run([sys.executable, WORKER, str(tmp_path), "0", "2", "solve", "1", "2000"],
                        capture_output=True, text=True, timeout=300)
    (tmp_path / "stop").write_text("1")
    idle.communicate(timeout=120)
    assert r0.returncode == 0, r0.stderr[-3000:]
    assert "ERR" in r0.stdout and "did not arrive" in r0.stdout, r0.stdout
