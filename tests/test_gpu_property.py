"""GPU parity on random shapes and layouts (hypothesis): the drawn cases of
tests/test_property_cpu.py, run through the C ABI on cuda:0 (every rank on one
GPU) and compared with the oracle byte for byte -- odd widths, partial fp8
blocks, ragged tails, KV replication, pipeline stages and DP replicas the
hand-written cases do not list."""
from __future__ import annotations

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings

import oracle
from tests import harness
from tests.test_property_cpu import case

pytestmark = pytest.mark.gpu


@settings(max_examples=200, deadline=None, suppress_health_check=list(HealthCheck), derandomize=True)
@given(case())
def test_random_layouts_gpu_vs_oracle(c):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_24034_b200 import build
    build.build()
    from paper_2505_24034_b200 import llrl as L
    m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg, _ = c
    O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg)
    if O.status != 0:
        return
    S, D = L.describe(m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg)
    ns, nd = S.n_ranks, D.n_ranks
    try:
        plan = L.Plan(S, D, [0] * ns, [0] * nd)
    except L.LlrlError as e:
        assert e.status == L.E_UNSUPPORTED and ddt in ("mxfp8", "mxfp4", "nvfp4")
        return
    src = harness.host_src(O, 7)
    want = harness.oracle_dst(O, src, 0x3C)
    dev = torch.device("cuda", 0)
    sb = [torch.from_numpy(b).to(dev) for b in src]
    db = [torch.full((D.rank_bytes(g),), 0x3C, dtype=torch.uint8, device=dev) for g in range(nd)]
    comm = L.Comm(0) if ddt == "nvfp4" else None
    stream = torch.cuda.current_stream(dev)
    for _ in range(2):                           # twice: device-side state resets between syncs
        plan.sync(comm, 0, [t.data_ptr() for t in sb], [t.data_ptr() for t in db], stream.cuda_stream)
    torch.cuda.synchronize()
    for g in range(nd):
        got = db[g].cpu().numpy()
        if not np.array_equal(got, want[g]):
            bad = np.nonzero(got != want[g])[0]
            raise AssertionError(f"{c}: dst rank {g}: {bad.size} bytes differ, first {bad[:8]}")
    if comm is not None:
        comm.close()
    plan.close()
