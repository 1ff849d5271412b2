"""bench.py's N-rank path on CPU: `torchrun --nproc-per-node 2 bench.py
--gpus 2 --dry-run` runs the same topology / workload / shard / record-fold /
max-over-ranks code as the GPU arm, over gloo, with synthetic per-candidate
outputs; the fold must equal the one-process fold bit for bit.  And
`bench.py --gpus N` without torchrun must refuse to run on fewer GPUs."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _last_json(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_two_ranks_dry_run_equals_one_process():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"),
           "--gpus", "2", "--dry-run"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    two = _last_json(r.stdout)
    one = _last_json(subprocess.run([sys.executable, str(ROOT / "bench.py"), "--dry-run",
                                     "--config", "c4"], capture_output=True, text=True,
                                    timeout=600, env=env, cwd=ROOT, check=True).stdout)
    assert two["mode"] == "ranks" and two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["workload"] == one["workload"] and two["workload"].startswith("c4: K=262144")
    assert two["scaling"] == "strong"
    assert two["shard0"] == [0, 131072]
    assert two["result_hex"] == one["result_hex"]


def test_gpus_flag_fails_loudly_without_the_gpus():
    import torch
    n = torch.cuda.device_count() + 1
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n)],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0
    assert f"--gpus {n}: needs {n} CUDA device(s)" in (r.stderr + r.stdout)


def test_torchrun_world_must_match_gpus_flag():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0 and "torchrun started 2 ranks" in (r.stderr + r.stdout)
