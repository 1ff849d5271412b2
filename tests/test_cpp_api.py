"""The C++ drop-in API (include/tmpc_b200/planner.hpp) compiled against the
reference's own headers (tests/cpp/test_planner_api.cpp)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "test_planner_api"
needs_bin = pytest.mark.skipif(not BIN.exists(), reason="C++ API test binary not built")


@needs_bin
def test_cpp_api_host_checks():
    import torch
    if torch.cuda.is_available():
        pytest.skip("host-only path expects no GPU")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "host checks ok" in r.stdout


@needs_bin
@pytest.mark.gpu
def test_cpp_api_solve_on_gpu():
    r = subprocess.run([str(BIN), "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "gpu checks ok" in r.stdout
