"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, bit-exact.

Small sizes (toy, several tiles and ragged tails): every byte of every
generator buffer.  Full BASELINE sizes, in the launch configuration bench.py
times (runner.SyncJob): every byte too, the oracle streamed per generator
parameter over the host cores, plus exact write coverage.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from synth import MODELS, CONFIGS, LayoutConfig
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


@pytest.fixture(params=["default", "tma"])
def cast_path(request, monkeypatch):
    """Toy syncs are tiny, so the product picks the register cast kernel for them
    (runtime.cu); run the toy cases through the TMA kernel the large syncs use as
    well."""
    if request.param == "tma":
        monkeypatch.setenv("LLRL_CAST_VARIANT", "6")
    return request.param


def _toy_job(rt, model_name, fsdp, tpt, tpg, sdt, ddt, inner=False, n_layers=None, dp=1, ppt=1, ppg=1):
    llrl, runner = rt
    cfg = LayoutConfig("t", model_name, fsdp, tpt, tpg, sdt, ddt, "colocated", inner, dp_gen=dp, pp_train=ppt,
                       pp_gen=ppg)
    return runner.SyncJob(runner.JobSpec(cfg, 1, n_layers=n_layers), fill=False)


def _run_and_compare(rt, job, seed, sentinel=0xA5, inject=None):
    cfg = job.cfg
    ol = oracle.Layout(job.model, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                       cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    src = harness.host_src(ol, seed)
    if inject is not None:
        inject(ol, src)
    for r, t in job.src.items():
        t.copy_(torch.from_numpy(src[r]))
    for g, t in job.dst.items():
        t.fill_(sentinel)
    job.sync()
    torch.cuda.synchronize()
    want = harness.oracle_dst(ol, src, sentinel)
    for g, t in job.dst.items():
        got = t.cpu().numpy()
        if not np.array_equal(got, want[g]):
            bad = np.nonzero(got != want[g])[0]
            raise AssertionError(f"dst rank {g}: {bad.size} bytes differ, first at {bad[:8]}")


def test_fill_matches_synth(rt):
    """K0 (CUDA) == synth (numpy) bit for bit: both sides use the same generator."""
    llrl, runner = rt
    for sdt in ("f32", "bf16"):
        job = _toy_job(rt, "toy", 3, 2, 4, sdt, "bf16")
        for t in job.src.values():
            t.zero_()                     # padding: the fill writes the pieces only (as host_src)
        job.fill(7)
        ol = oracle.Layout(job.model, 3, 2, 4, sdt, "bf16")
        want = harness.host_src(ol, 7)
        for r, t in job.src.items():
            assert np.array_equal(t.cpu().numpy(), want[r])
        job.close()


SWEEP = [(f, tt, tg, sdt, ddt) for f in (1, 2, 3, 8) for tt in (1, 2, 4) for tg in (1, 2, 4, 8)
         for sdt, ddt in (("f32", "bf16"), ("bf16", "fp8"), ("bf16", "mxfp8"), ("f32", "mxfp4"))]


@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt", SWEEP)
def test_toy_parity_sweep(rt, cast_path, fsdp, tpt, tpg, sdt, ddt):
    job = _toy_job(rt, "toy", fsdp, tpt, tpg, sdt, ddt)
    _run_and_compare(rt, job, seed=fsdp * 100 + tpt * 10 + tpg)
    job.close()


@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt", [
    (2, 1, 2, "f32", "bf16"), (2, 2, 8, "bf16", "fp8"), (3, 1, 4, "bf16", "nvfp4")])
def test_double_buffered_generator(rt, fsdp, tpt, tpg, sdt, ddt):
    """NEXT f3: with double buffering the sync writes the back set while the
    generator's front set stays untouched (a reader on another stream sees the
    previous weights throughout), and swap() publishes the new weights."""
    llrl, runner = rt
    cfg = LayoutConfig("t", "toy", fsdp, tpt, tpg, sdt, ddt, "colocated")
    job = runner.SyncJob(runner.JobSpec(cfg, 1), fill=False, double_buffer=True)
    ol = oracle.Layout(job.model, fsdp, tpt, tpg, sdt, ddt, False)
    for t in list(job.front.values()) + list(job.dst.values()):
        t.fill_(0x5A)
    reader = torch.cuda.Stream()
    prev = None
    for k in range(3):
        src = harness.host_src(ol, 40 + k)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        torch.cuda.synchronize()
        snap = {g: t.clone() for g, t in job.front.items()}
        reads = []
        with torch.cuda.stream(reader):           # the "generator" keeps reading its weights
            for _ in range(4):
                reads.append({g: t.clone() for g, t in job.front.items()})
        job.sync()
        torch.cuda.synchronize()
        for g, t in job.front.items():            # untouched by the sync
            assert torch.equal(t, snap[g]), f"sync {k} wrote the front buffer of rank {g}"
            assert all(torch.equal(rd[g], snap[g]) for rd in reads)
        job.swap()
        want = harness.oracle_dst(ol, src, 0x5A)
        for g, t in job.front.items():
            assert np.array_equal(t.cpu().numpy(), want[g]), f"sync {k}: front rank {g}"
        if prev is not None:
            for g in job.dst:                     # the next target is the older set
                assert job.dst[g].data_ptr() == prev[g]
        prev = {g: t.data_ptr() for g, t in job.front.items()}
    job.close()


@pytest.mark.parametrize("model,fsdp,tpt,tpg,sdt,ddt", [
    ("toy", 2, 1, 2, "f32", "bf16"),
    ("toy", 3, 1, 4, "f32", "fp8"),
    ("toy", 2, 2, 8, "bf16", "mxfp8"),
    ("toy", 3, 1, 4, "bf16", "mxfp4"),
    ("toy", 2, 2, 8, "bf16", "nvfp4"),
    ("ragged", 3, 1, 5, "f32", "bf16"),
    ("ragged", 7, 5, 1, "bf16", "fp8"),
    ("wide", 2, 2, 1, "bf16", "mxfp4"),
])
def test_guard_bands(rt, cast_path, model, fsdp, tpt, tpg, sdt, ddt):
    """Out-of-bounds check without compute-sanitizer (closed on this pool): every
    trainer and generator buffer sits inside a larger allocation between 64 KiB
    canary bands; after the sync the generator bytes match the oracle, no canary
    byte changed (no write before / after any buffer) and the trainer bytes are
    unchanged (the path only reads them)."""
    job = _toy_job(rt, model, fsdp, tpt, tpg, sdt, ddt)
    G = 1 << 16
    bigs = []

    def guarded(t, canary):
        big = torch.full((t.numel() + 2 * G,), canary, dtype=torch.uint8, device=t.device)
        bigs.append((big, t.numel(), canary))
        return big[G:G + t.numel()]

    job.src = {r: guarded(t, 0xC3) for r, t in job.src.items()}
    job.dst = {g: guarded(t, 0x3C) for g, t in job.dst.items()}
    job.src_ptrs = [job.src[r].data_ptr() if r in job.src else 0 for r in range(job.S.n_ranks)]
    job.dst_ptrs = [job.dst[g].data_ptr() if g in job.dst else 0 for g in range(job.D.n_ranks)]
    _run_and_compare(rt, job, seed=77)
    before = {r: t.cpu().numpy().copy() for r, t in job.src.items()}
    job.sync()
    torch.cuda.synchronize()
    for r, t in job.src.items():
        assert np.array_equal(t.cpu().numpy(), before[r]), f"trainer rank {r} modified"
    for big, n, canary in bigs:
        h = big.cpu().numpy()
        assert (h[:G] == canary).all() and (h[G + n:] == canary).all(), "write outside a rank buffer"
    job.close()


@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt,inner", [
    (2, 1, 2, "f32", "bf16", False),    # C1
    (3, 1, 4, "f32", "fp8", False),     # multi-source (pull) fp8 blocks
    (2, 2, 8, "bf16", "fp8", True),     # KV replication + FSDP-inner + multi-source blocks
    (3, 2, 4, "f32", "f32", False),     # identity (provenance mode)
    (8, 4, 8, "bf16", "bf16", False),   # 32 trainer ranks
    (1, 8, 8, "f32", "fp8", False),
    (3, 1, 4, "f32", "mxfp8", False),   # MXFP8 (R13)
    (2, 2, 8, "bf16", "mxfp8", True),
    (3, 1, 4, "bf16", "mxfp4", False),  # MXFP4 (R15)
    (2, 2, 8, "f32", "mxfp4", True),
    (2, 1, 2, "f32", "nvfp4", False),   # NVFP4 (R16): per-tensor amax over several trainer ranks
    (2, 2, 8, "bf16", "nvfp4", True),
    (3, 1, 4, "bf16", "nvfp4", False),
])
def test_toy_parity_odd(rt, cast_path, fsdp, tpt, tpg, sdt, ddt, inner):
    job = _toy_job(rt, "toy", fsdp, tpt, tpg, sdt, ddt, inner)
    _run_and_compare(rt, job, seed=9)
    job.close()


def _inject_specials(ol, src):
    """Ties, subnormals, +-0, near-overflow, huge values, fp8 outlier / zero blocks."""
    rng = np.random.default_rng(3)
    specials32 = np.array([0x3F808000, 0x3F818000, 0x00038000, 0x80008000, 0x00000001, 0x80000000,
                           0x00000000, 0x7F7F8000, 0x7F7FFFFF, 0xFF7F0000, 0x3F7FFFFF, 0x0080FFFF,
                           0x33800000, 0x007FFFFF, 0x477FE000, 0xC3E00000], np.uint32)
    for r, b in enumerate(src):
        if ol.src_dtype == "f32":
            w = b.view(np.uint32)
            idx = rng.integers(0, w.size, 4096)
            w[idx] = rng.choice(specials32, idx.size)
        else:
            w = b.view(np.uint16)
            idx = rng.integers(0, w.size, 4096)
            w[idx] = rng.choice((specials32 >> 16).astype(np.uint16), idx.size)
        # one all-zero stretch (an fp8 block of zeros when it lands in a linear weight)
        z = rng.integers(0, max(1, b.size - 70000))
        b[z:z + 65536] = 0


@pytest.mark.parametrize("sdt,ddt", [("f32", "bf16"), ("f32", "fp8"), ("bf16", "fp8"), ("bf16", "bf16"),
                                     ("f32", "mxfp8"), ("bf16", "mxfp8"), ("f32", "mxfp4"), ("bf16", "mxfp4"),
                                     ("f32", "nvfp4"), ("bf16", "nvfp4")])
def test_toy_parity_special_values(rt, cast_path, sdt, ddt):
    # tp_train = 1: no replicated trainer pieces, so injected values stay consistent
    job = _toy_job(rt, "toy", 3, 1, 4, sdt, ddt)
    _run_and_compare(rt, job, seed=5, inject=_inject_specials)
    job.close()


@pytest.mark.parametrize("fsdp,tpt,tpg,dp,sdt,ddt", [(4, 1, 1, 4, "f32", "bf16"), (2, 2, 2, 3, "bf16", "fp8")])
def test_toy_parity_generator_dp(rt, cast_path, fsdp, tpt, tpg, dp, sdt, ddt):
    """Generator DP replicas (R12) filled from the same trainer shards."""
    job = _toy_job(rt, "toy", fsdp, tpt, tpg, sdt, ddt, dp=dp)
    _run_and_compare(rt, job, seed=13)
    job.close()


@pytest.mark.parametrize("fsdp,tpt,ppt,tpg,ppg,dp,sdt,ddt", [
    (2, 1, 2, 2, 1, 1, "f32", "bf16"), (1, 2, 1, 2, 2, 1, "bf16", "fp8"), (3, 1, 2, 4, 2, 2, "f32", "mxfp8")])
def test_toy_parity_pipeline_stages(rt, cast_path, fsdp, tpt, ppt, tpg, ppg, dp, sdt, ddt):
    """Decoupled pipeline parallelism (R14), with and without DP replicas."""
    job = _toy_job(rt, "toy", fsdp, tpt, tpg, sdt, ddt, dp=dp, ppt=ppt, ppg=ppg)
    _run_and_compare(rt, job, seed=17)
    job.close()


@pytest.mark.parametrize("model,fsdp,tpt,tpg,sdt,ddt", [
    ("ragged", 3, 1, 5, "f32", "bf16"), ("ragged", 7, 5, 1, "bf16", "fp8"), ("ragged", 2, 1, 5, "f32", "f32"),
    ("ragged", 3, 1, 5, "bf16", "fp8"),
    ("wide", 2, 2, 1, "f32", "bf16"), ("wide", 3, 1, 2, "bf16", "fp8"), ("wide", 1, 2, 1, "f32", "mxfp8"),
    ("wide", 2, 2, 1, "bf16", "mxfp4"), ("head_only", 3, 2, 4, "f32", "bf16"), ("toy", 32, 1, 2, "f32", "bf16")])
def test_edge_shapes_parity(rt, cast_path, model, fsdp, tpt, tpg, sdt, ddt):
    """Scalar fallbacks (no dimension a multiple of 8), partial fp8 blocks,
    rows wider than a TMA stage, a model without decoder layers, and trainer
    ranks holding nothing (FSDP 32 over 8-row norms)."""
    job = _toy_job(rt, model, fsdp, tpt, tpg, sdt, ddt)
    _run_and_compare(rt, job, seed=23)
    job.close()


def test_toy_parity_repeated_syncs(rt):
    """The same plan run many times (epoch counters, no stale state)."""
    job = _toy_job(rt, "toy", 4, 1, 4, "f32", "bf16")
    for i in range(5):
        _run_and_compare(rt, job, seed=20 + i, sentinel=i)
    job.close()


# ---------------------------------------------------------------- full sizes
#
# Every byte of every generator buffer at BASELINE sizes, in the launch
# configuration bench.py times (runner.spec_for(name, 1) -> SyncJob, all ranks
# on GPU 0): trainer buffers filled by the input generator at the ORACLE's
# offsets, the oracle streamed one generator parameter at a time on the host
# cores, plus exact write coverage (tests/harness.py: full_parity).


def _full_parity(rt, name, n_layers=None):
    llrl, runner = rt
    spec = runner.spec_for(name, 1)
    if n_layers is not None:
        spec = runner.JobSpec(spec.cfg, 1, n_layers=n_layers)
    job = runner.SyncJob(spec, seed=0, fill=False)
    cfg = job.cfg
    ol = oracle.Layout(job.model, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                       cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    try:
        t = harness.full_parity(ol, job)
    finally:
        job.close()
        torch.cuda.empty_cache()
    print(f"{name} ({job.model.n_layers} layers): {t}")


def test_full_c2_8b_every_byte(rt):
    """C2 (Llama-3.1 8B fp32 FSDP=4 -> bf16 TP=4), the whole model, as bench.py runs it."""
    _full_parity(rt, "c2")


@pytest.mark.parametrize("name,layers", [("c3", None), ("c4", None), ("c7", 8), ("c10", 8), ("c11", 8),
                                         ("c12", 8)])
def test_full_70b_every_byte(rt, name, layers):
    """The 70B configurations at G=1 with embed and lm_head: C3 (bf16
    FSDP8->TP8) and C4 (fp8 blocks) on the 40-layer slice bench.py times; C7
    MXFP8, C10 MXFP4, C11 NVFP4 and C12 NVFP4 from FSDP chunks (strided tiles,
    cross-chunk amax) on 8 decoder layers to bound the suite's time (the same
    kernels and launch configuration; all six at 40 layers:
    profiles/r02/gpu_full_parity_every_byte_40L.log)."""
    _full_parity(rt, name, n_layers=layers)


def test_full_c5_405b_slice_every_byte(rt):
    """C5 (405B layer slice, bf16 FSDP=2 x TP=4 -> TP=8, TP-innermost mesh): two
    of its 16 layers on one GPU (the 16-layer slice needs 2+ GPUs)."""
    _full_parity(rt, "c5", n_layers=2)


@pytest.mark.parametrize("variant", range(9))
def test_toy_parity_cast_variants(rt, variant, monkeypatch):
    """Every cast-kernel variant (LLRL_CAST_VARIANT tuning knob) is bit-exact."""
    monkeypatch.setenv("LLRL_CAST_VARIANT", str(variant))
    for sdt, ddt, f, tt, tg in (("f32", "bf16", 3, 2, 4), ("bf16", "bf16", 8, 1, 8), ("f32", "f32", 2, 1, 2)):
        job = _toy_job(rt, "toy", f, tt, tg, sdt, ddt)
        _run_and_compare(rt, job, seed=variant)
        job.close()


@pytest.mark.parametrize("tmap", ["0", "1"])
@pytest.mark.parametrize("frac", ["0", "0.5", "1"])
@pytest.mark.parametrize("block", ["0", "1"])
def test_toy_parity_cast_item_order(rt, tmap, frac, block, monkeypatch):
    """The TMA cast launch's item orders (LLRL_STATIC_FRAC: static share, rest
    claimed from the queue; LLRL_STATIC_BLOCK: static items striped or one block
    per CTA) and its optional 3-D tensor-map boxes for strided sources
    (LLRL_CAST_TMAP=1: o / down column bands of FSDP row chunks) are bit-exact,
    for every cast flavour (bf16, f32, MXFP8, NVFP4)."""
    monkeypatch.setenv("LLRL_STATIC_FRAC", frac)
    monkeypatch.setenv("LLRL_STATIC_BLOCK", block)
    monkeypatch.setenv("LLRL_CAST_TMAP", tmap)
    for sdt, ddt, f, tt, tg in (("f32", "bf16", 3, 1, 4), ("bf16", "bf16", 4, 1, 2), ("f32", "f32", 2, 1, 2),
                                ("bf16", "mxfp8", 4, 1, 4), ("f32", "nvfp4", 2, 1, 4)):
        job = _toy_job(rt, "toy", f, tt, tg, sdt, ddt)
        _run_and_compare(rt, job, seed=7)
        job.close()


@pytest.mark.parametrize("run", ["0", "1", "7", "32"])
def test_toy_parity_nv_amax_runs(rt, run, monkeypatch):
    """NVFP4 amax pass with its items split into runs striped over the CTAs
    (LLRL_NV_RUN; 0 = one range per CTA, the default): bit-exact, including
    tensors whose items are spread over many CTAs (per-tensor amax combined by
    atomicMax)."""
    monkeypatch.setenv("LLRL_NV_RUN", run)
    for sdt, f, tt, tg in (("bf16", 2, 2, 8), ("f32", 3, 1, 4), ("bf16", 8, 1, 8)):
        job = _toy_job(rt, "toy", f, tt, tg, sdt, "nvfp4")
        _run_and_compare(rt, job, seed=int(run) + 5)
        job.close()


@pytest.mark.parametrize("variant", ["6", "7"])
@pytest.mark.parametrize("frac", ["0", "1"])
def test_long_items_claimed_phase(rt, variant, frac):
    """Items of many more stages than the ring holds (LLRL_CHUNK_ELEMS = 128 Ki
    elements: up to 32 stages), claimed or static, in a fresh process
    (tests/long_items_worker.py): every generator byte equals the oracle's.
    Guards the claimed phase's hand-off (a consumer must keep its own copy of
    the item: the producer recycles the item's first stage while the consumer
    is still on later chunks)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LLRL_CHUNK_ELEMS="131072", LLRL_STATIC_FRAC=frac, LLRL_CAST_VARIANT=variant)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "long_items_worker.py")], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "LONG_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_toy_parity_fp8_variants(rt, variant, monkeypatch):
    """Both fp8 kernels (register / TMA-pipelined, LLRL_FP8_VARIANT) are bit-exact,
    including multi-source (pull) blocks and partial edge blocks."""
    monkeypatch.setenv("LLRL_FP8_VARIANT", str(variant))
    for sdt, f, tt, tg in (("bf16", 1, 8, 8), ("f32", 3, 1, 4), ("bf16", 2, 2, 8), ("f32", 2, 1, 2)):
        job = _toy_job(rt, "toy", f, tt, tg, sdt, "fp8")
        _run_and_compare(rt, job, seed=40 + variant)
        job.close()


@pytest.mark.parametrize("sdt,ddt,f,tt,tg", [("f32", "bf16", 2, 1, 2), ("bf16", "fp8", 2, 2, 8), ("f32", "fp8", 3, 1, 4)])
def test_toy_parity_sync_group(rt, sdt, ddt, f, tt, tg):
    """llrl_sync_group over every layer group (in reverse order) == the whole sync."""
    job = _toy_job(rt, "toy", f, tt, tg, sdt, ddt)
    ol = oracle.Layout(job.model, f, tt, tg, sdt, ddt)
    src = harness.host_src(ol, 77)
    for r, t in job.src.items():
        t.copy_(torch.from_numpy(src[r]))
    for t in job.dst.values():
        t.fill_(0x33)
    n = job.plan.num_groups()
    assert n == job.model.n_layers + 2
    for grp in reversed(range(n)):
        job.plan.sync_group(job.comm, job.device, grp, job.src_ptrs, job.dst_ptrs, job.stream.cuda_stream)
    torch.cuda.synchronize()
    want = harness.oracle_dst(ol, src, 0x33)
    for g, t in job.dst.items():
        assert np.array_equal(t.cpu().numpy(), want[g]), g
    job.close()


@pytest.mark.parametrize("sdt,ddt", [("f32", "bf16"), ("bf16", "fp8")])
def test_toy_parity_overlapped_step(rt, sdt, ddt):
    """f3: per-layer optimizer pass (x * 1.0, values unchanged) overlapped with
    llrl_sync_group streaming the previous layer == the plain sync."""
    job = _toy_job(rt, "toy", 2, 2, 4, sdt, ddt)
    ol = oracle.Layout(job.model, 2, 2, 4, sdt, ddt)
    src = harness.host_src(ol, 55)
    for r, t in job.src.items():
        t.copy_(torch.from_numpy(src[r]))
    for t in job.dst.values():
        t.fill_(0x21)
    opt_stream = torch.cuda.Stream()
    job.overlapped_step(lambda vs: [v.mul_(1.0) for v in vs], opt_stream)
    torch.cuda.synchronize()
    want = harness.oracle_dst(ol, src, 0x21)
    for g, t in job.dst.items():
        assert np.array_equal(t.cpu().numpy(), want[g]), g
    job.close()


@pytest.mark.parametrize("sdt,ddt", [("f32", "bf16"), ("bf16", "fp8"), ("bf16", "mxfp8")])
@pytest.mark.parametrize("kernel", ["default", "tma-claimed"])
def test_toy_parity_cuda_graph_replay(rt, sdt, ddt, kernel, monkeypatch):
    """Completion state lives on the device, so a warmed-up sync (and the per-layer
    overlapped step) can be captured once in a CUDA graph and replayed -- also
    through the TMA cast kernel with every item claimed from its queue (the last
    CTA out resets the queue for the next launch / replay)."""
    if kernel == "tma-claimed":
        monkeypatch.setenv("LLRL_CAST_VARIANT", "6")
        monkeypatch.setenv("LLRL_STATIC_FRAC", "0")
    job = _toy_job(rt, "toy", 2, 2, 4, sdt, ddt)
    ol = oracle.Layout(job.model, 2, 2, 4, sdt, ddt)
    job.sync()                                   # warm-up: uploads tables, encodes tensor maps
    torch.cuda.synchronize()
    g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    opt_stream = torch.cuda.Stream()
    with torch.cuda.graph(g1):
        job.sync(stream=torch.cuda.current_stream())
    with torch.cuda.graph(g2):
        job.overlapped_step(lambda vs: [v.mul_(1.0) for v in vs], opt_stream, stream=torch.cuda.current_stream())
    for rep, g in enumerate((g1, g2, g1, g2)):
        src = harness.host_src(ol, 70 + rep)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x3C)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        want = harness.oracle_dst(ol, src, 0x3C)
        for q, t in job.dst.items():
            assert np.array_equal(t.cpu().numpy(), want[q]), (rep, q)
    job.close()


@pytest.mark.parametrize("sdt,f,tt,tg", [("bf16", 2, 2, 8), ("f32", 3, 1, 4)])
def test_toy_parity_cuda_graph_replay_nvfp4(rt, sdt, f, tt, tg):
    """NVFP4 sync captured in a CUDA graph: the amax handshake (memset, amax,
    scale, fetch kernels, waits) and the quantising cast replay with new
    trainer values each time (tensor amax and scales change)."""
    job = _toy_job(rt, "toy", f, tt, tg, sdt, "nvfp4")
    ol = oracle.Layout(job.model, f, tt, tg, sdt, "nvfp4")
    job.sync()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        job.sync(stream=torch.cuda.current_stream())
    for rep in range(3):
        src = harness.host_src(ol, 90 + rep)
        if rep >= 1:      # halve layer 0's q shard on trainer rank 0: its tensor amax drops,
            off, r0, r1, c0, c1 = ol.src_piece(0, 2)     # so a stale (not reset) amax would show
            n = (r1 - r0) * (c1 - c0)
            if sdt == "f32":
                x = src[0][off:off + 4 * n].view(np.float32)
                x *= np.float32(0.5)
            else:
                x = src[0][off:off + 2 * n].view(np.uint16)
                e = (x >> 7) & 0xFF
                x[e > 1] -= np.uint16(0x80)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x3C)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        want = harness.oracle_dst(ol, src, 0x3C)
        for q, t in job.dst.items():
            assert np.array_equal(t.cpu().numpy(), want[q]), (rep, q)
    job.close()


@pytest.mark.parametrize("sdt,ddt,f,tt,tg", [("f32", "bf16", 2, 1, 2), ("bf16", "fp8", 2, 2, 8),
                                           ("bf16", "mxfp8", 2, 2, 8), ("bf16", "mxfp4", 2, 2, 8),
                                           ("bf16", "nvfp4", 2, 2, 8), ("f32", "nvfp4", 3, 1, 4)])
def test_toy_parity_sync_host(rt, sdt, ddt, f, tt, tg):
    """llrl_sync_host: pinned host trainer shards in, host generator shards out,
    pipelined per layer group; twice, to exercise stream/event reuse."""
    job = _toy_job(rt, "toy", f, tt, tg, sdt, ddt)
    ol = oracle.Layout(job.model, f, tt, tg, sdt, ddt)
    for rep in range(2):
        src = harness.host_src(ol, 90 + rep)
        hs = {r: torch.from_numpy(src[r]).pin_memory() for r in job.src}
        hd = {g: torch.full((job.D.rank_bytes(g),), 0x44, dtype=torch.uint8).pin_memory() for g in job.dst}
        for t in job.src.values():
            t.fill_(0)                # the device copy must come from the host buffers
        for t in job.dst.values():
            t.fill_(0x44)             # padding inside a group's range travels back too
        job.sync_host(hs, hd)
        torch.cuda.synchronize()
        want = harness.oracle_dst(ol, src, 0x44)
        for g in job.dst:
            assert np.array_equal(hd[g].numpy(), want[g]), (rep, g)
    job.close()


@pytest.mark.parametrize("max_ctas", [1, 3, 64])
def test_toy_parity_capped_grid(rt, max_ctas):
    """llrl_plan_set_max_ctas: a capped grid (down to one CTA) still covers every item."""
    for sdt, ddt in (("f32", "bf16"), ("bf16", "fp8"), ("bf16", "mxfp4")):
        job = _toy_job(rt, "toy", 3, 2, 4, sdt, ddt)
        job.plan.set_max_ctas(job.device, max_ctas)
        _run_and_compare(rt, job, seed=max_ctas)
        job.close()
