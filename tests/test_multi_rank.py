"""Multi-rank planning cycle on CPU (gloo, world_size 2): each rank evaluates
its contiguous candidate shard (PL.shard_range) — here with the CPU oracle
standing in for the per-GPU kernel — reduces it to the product's per-GPU
record (tmpc_make_record, the host mirror of the kernel's reduction), one
all-gather of the records (the collective the device path issues as
ncclAllGather) and the product's fold (tmpc_fold_records, rank order)
select the global winner.  The result must equal the single-process solve
bit for bit for any world size: candidates draw controls from their GLOBAL
index and every reduction is order-independent."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_2603_20525_b200 import _abi, planner as PL
    from parity_util import problem

    w, p, smp_full, terr, keep = problem("c1", 512, 20)
    k0, kc = PL.shard_range(smp_full.k_count, rank, world)
    smp, keep2 = PL.make_sampling(w.cfg.__class__(**{**w.cfg.__dict__, "n_samples": 512}), k0, kc)
    smp.seed = smp_full.seed
    rc, res, cost, flags, margin, sub, err = Oracle("port").solve(p, smp, terr, w.s0, threads=2)
    assert rc == 0, err
    rec = PL.make_record(cost, flags, margin, k0, p.selection, sub)
    gathered = [None] * world
    dist.all_gather_object(gathered, PL.record_bytes(rec))
    res = PL.fold_records([PL.record_from_bytes(b) for b in gathered])
    if rank == 0:
        out.put(bytes(res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_argmin_equals_single_process(world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from oracle.oracle import Oracle
    from parity_util import problem, runner_up_gap

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    got = q.get(timeout=10)
    from paper_2603_20525_b200 import _abi, planner as PL

    w, p, smp, terr, keep = problem("c1", 512, 20)
    rc, res, cost, flags, margin, sub, err = Oracle("port").solve(p, smp, terr, w.s0, threads=4)
    one = PL.fold_records([PL.make_record(cost, flags, margin, 0, p.selection, sub)])
    assert got == bytes(one)  # bit-identical fold for world 1 and world 2
    r = _abi.tmpc_result.from_buffer_copy(got)
    assert r.best_index == res.best_index and r.best_cost == res.best_cost
    assert r.n_feasible == int((flags & 1).sum()) and r.n_candidates == 512
