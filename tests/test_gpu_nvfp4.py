"""NVFP4 (reading R16) extras on the GPU, bit-exact against the oracle:
the one-pass sync with a caller-supplied per-tensor amax (llrl_sync_nv_amax,
verdict r1 #3), amax-table regions per plan on a shared comm and the
library-owned comm of a one-GPU NVFP4 plan called with comm=NULL."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from synth import LayoutConfig
from tests import harness

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_24034_b200 import build
    build.build()
    from paper_2505_24034_b200 import llrl, runner
    return llrl, runner


def _job(rt, fsdp, tpt, tpg, sdt, model="toy", n_layers=None):
    llrl, runner = rt
    cfg = LayoutConfig("t", model, fsdp, tpt, tpg, sdt, "nvfp4", "colocated")
    return runner.SyncJob(runner.JobSpec(cfg, 1, n_layers=n_layers), fill=False)


def _ol(job):
    c = job.cfg
    return oracle.Layout(job.model, c.fsdp, c.tp_train, c.tp_gen, c.src_dtype, c.dst_dtype)


@pytest.mark.parametrize("variant", ["default", "6"])
@pytest.mark.parametrize("sdt,f,tt,tg", [("bf16", 2, 2, 8), ("f32", 3, 1, 4), ("bf16", 1, 2, 2)])
def test_toy_parity_nvfp4_supplied_amax(rt, monkeypatch, variant, sdt, f, tt, tg):
    """llrl_sync_nv_amax is byte-identical to the oracle with the caller's exact
    amax (computed here from the regions llrl_plan_nv_tensor_sources lists),
    eagerly and under CUDA-graph replay with new trainer values."""
    if variant != "default":
        monkeypatch.setenv("LLRL_CAST_VARIANT", variant)
    job = _job(rt, f, tt, tg, sdt)
    ol = _ol(job)
    assert job.plan.nv_num_tensors() == sum(ol.dst_param(q, gp)[2] for q in range(ol.n_dst)
                                            for gp in range(ol.n_dst_params))
    amax = torch.zeros(job.plan.nv_num_tensors(), dtype=torch.float32, device="cuda")
    graph = None
    for rep in range(4):
        src = harness.host_src(ol, 70 + rep)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x3C)
        amax.copy_(harness.caller_nv_amax(job))
        torch.cuda.synchronize()
        if graph is None:
            job.sync_nv_amax(amax)
        else:
            graph.replay()
        torch.cuda.synchronize()
        want = harness.oracle_dst(ol, src, 0x3C)
        for q, t in job.dst.items():
            assert np.array_equal(t.cpu().numpy(), want[q]), (rep, q)
        if rep == 1:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                job.sync_nv_amax(amax, stream=torch.cuda.current_stream())
    job.close()


def test_nv_tensor_sources_cover_each_tensor(rt):
    """The regions of each tensor hold exactly its generator-local element count."""
    job = _job(rt, 3, 2, 4, "bf16")
    ol = _ol(job)
    for tid in range(job.plan.nv_num_tensors()):
        t = job.plan.nv_tensor(tid)
        R, C, q = ol.dst_param(t.dst_rank, t.dst_param)[:3]
        assert q and t.device == 0
        assert sum(s.rows * s.cols for s in job.plan.nv_tensor_sources(tid)) == R * C
    job.close()


def test_nvfp4_plans_share_a_comm_and_null_comm(rt):
    """Two NVFP4 plans synced through one comm (interleaved, twice) each get
    their own amax-table region; a one-GPU NVFP4 sync with comm=NULL uses a
    library-owned comm."""
    jobs = [_job(rt, 2, 2, 8, "bf16"), _job(rt, 3, 1, 4, "f32")]
    comm = jobs[0].comm
    ols = [_ol(j) for j in jobs]
    s = torch.cuda.current_stream().cuda_stream
    for rep in range(2):
        srcs = [harness.host_src(ol, 30 + rep + 5 * k) for k, ol in enumerate(ols)]
        for j, src in zip(jobs, srcs):
            for r, t in j.src.items():
                t.copy_(torch.from_numpy(src[r]))
            for t in j.dst.values():
                t.fill_(0x11)
        for j in jobs:
            j.plan.sync(comm, 0, j.src_ptrs, j.dst_ptrs, s)
        torch.cuda.synchronize()
        for j, ol, src in zip(jobs, ols, srcs):
            want = harness.oracle_dst(ol, src, 0x11)
            for q, t in j.dst.items():
                assert np.array_equal(t.cpu().numpy(), want[q]), (rep, q)
    j, ol = jobs[1], ols[1]
    src = harness.host_src(ol, 36)
    for r, t in j.src.items():
        t.copy_(torch.from_numpy(src[r]))
    for t in j.dst.values():
        t.fill_(0x22)
    for _ in range(2):
        j.plan.sync(None, 0, j.src_ptrs, j.dst_ptrs, s)
    torch.cuda.synchronize()
    want = harness.oracle_dst(ol, src, 0x22)
    for q, t in j.dst.items():
        assert np.array_equal(t.cpu().numpy(), want[q]), q
    for j in jobs:
        j.close()


def test_full_c11_supplied_amax_every_byte(rt):
    """C11 (70B bf16 TP=8 -> NVFP4 TP=8) at G=1 through llrl_sync_nv_amax, 8
    decoder layers + embed / lm_head, every byte against the oracle (streamed)."""
    llrl, runner = rt
    spec = runner.spec_for("c11", 1)
    job = runner.SyncJob(runner.JobSpec(spec.cfg, 1, n_layers=8), seed=0, fill=False)
    ol = _ol(job)
    try:
        harness.fill_src_device(ol, 0, job.src)
        amax = harness.caller_nv_amax(job)
        for t in job.dst.values():
            t.fill_(0xA5)
        job.sync_nv_amax(amax)
        torch.cuda.synchronize()
        harness.streamed_compare(ol, 0, job.dst, 0xA5)
    finally:
        job.close()
