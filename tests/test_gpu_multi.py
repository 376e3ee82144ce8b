"""Multi-GPU parity (one process per GPU over NVLink): runs tests/mp_worker.py
under torchrun on 2 (and, when present, 4 / 8) GPUs.  Skipped with < 2 GPUs."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n, full, port, extra=(), env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mp_worker.py")]
    if full:
        cmd.append("--full")
    cmd += list(extra)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200,
                       env=dict(os.environ, **(env or {})))
    assert r.returncode == 0 and "MP_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-5000:]


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_parity(n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    _run(n, full=(n == max(k for k in (2, 4, 8) if k <= torch.cuda.device_count())), port=29500 + n)


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("mode", ["split", "tma"])
def test_multicast_opt_in_paths_parity(n, mode):
    """The opt-in multicast paths are bit-exact: the egress split
    (LLRL_MC_UNICAST_PERIOD=k: every k-th multicast item pushed to each replica
    as plain peer stores) and the TMA cast kernel feeding NVLS through its bulk
    storer (LLRL_MC_TMA=1)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    env = {"LLRL_MC_UNICAST_PERIOD": "3"} if mode == "split" else {"LLRL_MC_TMA": "1"}
    _run(n, full=False, port=29520 + n + (10 if mode == "tma" else 0), extra=["--mc-only"], env=env)
