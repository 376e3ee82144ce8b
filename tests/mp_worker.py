"""Multi-GPU parity worker (one process per GPU), launched by
tests/test_gpu_multi.py as

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      --master-port P tests/mp_worker.py [--full]

Each rank owns the trainer / generator ranks placed on its GPU, maps its
peers' buffers over IPC, runs llrl_sync (push over NVLink + completion flags)
and compares every generator buffer it owns with the CPU oracle, byte for byte
(toy and, with --full, every full-size config: streamed per generator
parameter, tests/harness.py).
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
from synth import LayoutConfig  # noqa: E402
from tests import harness  # noqa: E402


def toy_case(runner, world, fsdp, tpt, tpg, sdt, ddt, placement, inner=False, seed=3, reps=2, dp=1, ppt=1, ppg=1,
             multicast=False):
    cfg = LayoutConfig("mp", "toy", fsdp, tpt, tpg, sdt, ddt, placement, inner, dp_gen=dp, pp_train=ppt, pp_gen=ppg)
    job = runner.SyncJob(runner.JobSpec(cfg, world), fill=False, multicast=multicast)
    if multicast:
        assert job.mc_positions()[0], "expected multicast-eligible replicas"
    ol = oracle.Layout(job.model, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg)
    for rep in range(reps):
        src = harness.host_src(ol, seed + rep)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x5A)
        torch.cuda.synchronize()
        dist.barrier()
        job.sync()
        torch.cuda.synchronize()
        dist.barrier()
        want = harness.oracle_dst(ol, src, 0x5A)
        for g, t in job.dst.items():
            got = t.cpu().numpy()
            if not np.array_equal(got, want[g]):
                bad = np.nonzero(got != want[g])[0]
                raise AssertionError(f"{cfg} rep {rep}: dst rank {g} differs at {bad.size} bytes, first {bad[:6]}")
    # layer-group streaming across GPUs (not NVFP4: a tensor's scale needs its whole amax, R16)
    if ddt != "nvfp4":
        src = harness.host_src(ol, seed + 50)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x5A)
        torch.cuda.synchronize()
        dist.barrier()
        for grp in range(job.plan.num_groups()):
            job.plan.sync_group(job.comm, job.device, grp, job.src_ptrs, job.dst_ptrs, job.stream.cuda_stream)
        torch.cuda.synchronize()
        dist.barrier()
        want = harness.oracle_dst(ol, src, 0x5A)
        for g, t in job.dst.items():
            assert np.array_equal(t.cpu().numpy(), want[g]), f"{cfg} sync_group: dst rank {g}"
    # the host-buffer entry (NVFP4: whole buffers in, whole sync, whole buffers out)
    src = harness.host_src(ol, seed + 60)
    hs = {r: torch.from_numpy(src[r]).pin_memory() for r in job.src}
    hd = {g: torch.full((job.D.rank_bytes(g),), 0x5A, dtype=torch.uint8).pin_memory() for g in job.dst}
    dist.barrier()
    job.sync_host(hs, hd)
    torch.cuda.synchronize()
    dist.barrier()
    want = harness.oracle_dst(ol, src, 0x5A)
    for g in job.dst:
        assert np.array_equal(hd[g].numpy(), want[g]), f"{cfg} sync_host: dst rank {g}"
    assert job.comm is None or not job.comm.timed_out()
    # CUDA-graph replay of the multi-GPU sync (device-side completion state)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        job.sync(stream=torch.cuda.current_stream())
    for rep in range(2):
        src = harness.host_src(ol, seed + 80 + rep)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x5A)
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        dist.barrier()
        want = harness.oracle_dst(ol, src, 0x5A)
        for q, t in job.dst.items():
            assert np.array_equal(t.cpu().numpy(), want[q]), f"{cfg} graph replay {rep}: dst rank {q}"
    job.close()


def nccl_replica_case(runner, world, fsdp, tpt, tpg, sdt, ddt, dp, seed=21, mode=1):
    """a5 through llrl_sync on an LLRL_PLAN_NCCL plan: mode 1 = replica 0 by the
    fused kernels, replicas 1.. by ncclBroadcast (R17); mode 2 = FSDP chunks
    ncclAllGather-ed into every replica, no kernel of ours (R18)."""
    cfg = LayoutConfig("mp", "toy", fsdp, tpt, tpg, sdt, ddt, "colocated", dp_gen=dp)
    job = runner.SyncJob(runner.JobSpec(cfg, world), fill=False, replicate="nccl")
    info = job.plan.nccl_info(job.device)
    assert info.mode == mode, (cfg, info.mode)
    if mode == 2:
        assert job.plan.stats().n_items == 0 and info.n_allgathers > 0
    ol = oracle.Layout(job.model, fsdp, tpt, tpg, sdt, ddt, False, dp)
    for rep in range(2):
        src = harness.host_src(ol, seed + rep)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x5A)
        torch.cuda.synchronize()
        dist.barrier()
        job.sync()
        torch.cuda.synchronize()
        dist.barrier()
        want = harness.oracle_dst(ol, src, 0x5A)
        for g, t in job.dst.items():
            assert np.array_equal(t.cpu().numpy(), want[g]), f"{cfg} nccl replicate rep {rep}: dst rank {g}"
    job.close()


def double_buffer_case(runner, world, fsdp, tpt, tpg, sdt, ddt, placement, seed=31):
    """f3 across GPUs: peers push into the back set (both sets IPC-mapped), the
    front set is untouched until every process swaps."""
    cfg = LayoutConfig("mp", "toy", fsdp, tpt, tpg, sdt, ddt, placement)
    job = runner.SyncJob(runner.JobSpec(cfg, world), fill=False, double_buffer=True)
    ol = oracle.Layout(job.model, fsdp, tpt, tpg, sdt, ddt, False)
    for t in list(job.front.values()) + list(job.dst.values()):
        t.fill_(0x5A)
    old = harness.oracle_dst(ol, harness.host_src(ol, seed - 1), 0x5A)
    first = True
    for rep in range(3):
        src = harness.host_src(ol, seed + rep)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        torch.cuda.synchronize()
        snap = {g: t.cpu().numpy().copy() for g, t in job.front.items()}
        dist.barrier()
        job.sync()
        torch.cuda.synchronize()
        dist.barrier()
        for g, t in job.front.items():
            assert np.array_equal(t.cpu().numpy(), snap[g]), f"{cfg} rep {rep}: front rank {g} written"
            if not first:
                assert np.array_equal(snap[g], old[g])
        job.swap()
        first = False
        want = harness.oracle_dst(ol, src, 0x5A)
        for g, t in job.front.items():
            assert np.array_equal(t.cpu().numpy(), want[g]), f"{cfg} rep {rep}: dst rank {g}"
        old = want
    job.close()


def random_cases(runner, world, n=24, seed=2505):
    """Seeded random shapes and layouts (the same draws on every rank), each
    through llrl_sync across the GPUs twice and compared with the oracle byte
    for byte; invalid draws are skipped the same way on every rank."""
    from synth import MODELS
    from synth.configs import Model
    rng = np.random.default_rng(seed)
    ran = 0
    for i in range(400):
        if ran >= n:
            break
        ddt_s = [("f32", "bf16"), ("bf16", "bf16"), ("f32", "f32"), ("bf16", "fp8"), ("f32", "fp8"),
                 ("bf16", "mxfp8"), ("f32", "mxfp4"), ("bf16", "nvfp4")]
        sdt, ddt = ddt_s[rng.integers(len(ddt_s))]
        tpt = int(rng.choice([1, 2, 3, 4]))
        tpg = int(rng.choice([1, 2, 4, 8]))
        unit = tpt * tpg // int(np.gcd(tpt, tpg))
        if ddt in ("mxfp8", "mxfp4", "nvfp4"):
            unit *= 32
        kv = int(rng.choice(sorted({1, 2, 4, tpg})))
        m = Model(int(rng.integers(1, 3)), unit * int(rng.choice([1, 2])) * 8, kv * int(rng.choice([1, 2, unit])),
                  kv, int(rng.choice([8, 16, 32])), unit * int(rng.choice([8, 12])), unit * int(rng.choice([4, 6])),
                  int(rng.integers(0, 2)))
        d, q, k = m.d_model, m.n_heads * m.head_dim, m.n_kv_heads * m.head_dim
        if m.n_layers * (d * (q + 2 * k) + q * d + 3 * d * m.d_ffn) + 2 * m.vocab * d > 3_000_000:
            continue
        fsdp = int(rng.integers(1, 5))
        inner = bool(rng.integers(0, 2))
        dp, ppt, ppg = (int(rng.choice([1, 1, 2])) for _ in range(3))
        placement = str(rng.choice(["colocated", "rotated", "disjoint"]))
        O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg)
        if O.status != 0:
            continue
        name = f"rnd{i}"
        MODELS[name] = m
        cfg = LayoutConfig(name, name, fsdp, tpt, tpg, sdt, ddt, placement, inner, dp_gen=dp, pp_train=ppt,
                           pp_gen=ppg)
        try:
            job = runner.SyncJob(runner.JobSpec(cfg, world), fill=False)
        except Exception as e:           # tiles splitting a 1x32 / 1x16 group: UNSUPPORTED (R13, R16)
            assert "UNSUPPORTED" in str(e) or "status -4" in str(e), e
            dist.barrier()
            continue
        src = harness.host_src(O, 11 + i)
        want = harness.oracle_dst(O, src, 0x5A)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for t in job.dst.values():
            t.fill_(0x5A)
        torch.cuda.synchronize()
        dist.barrier()
        for _ in range(2):
            job.sync()
        torch.cuda.synchronize()
        dist.barrier()
        for g, t in job.dst.items():
            got = t.cpu().numpy()
            if not np.array_equal(got, want[g]):
                bad = np.nonzero(got != want[g])[0]
                raise AssertionError(f"random case {i} {m} {cfg}: dst rank {g}: {bad.size} bytes, first {bad[:6]}")
        if ddt != "nvfp4":                 # layer-group streaming (not NVFP4, R16)
            for t in job.dst.values():
                t.fill_(0x5A)
            torch.cuda.synchronize()
            dist.barrier()
            for grp in range(job.plan.num_groups()):
                job.sync_group(grp)
            torch.cuda.synchronize()
            dist.barrier()
            for g, t in job.dst.items():
                assert np.array_equal(t.cpu().numpy(), want[g]), f"random case {i} {cfg}: sync_group rank {g}"
        if True:                           # the host-buffer pipeline
            hs = {r: torch.from_numpy(src[r]).pin_memory() for r in job.src}
            hd = {g: torch.full((job.D.rank_bytes(g),), 0x5A, dtype=torch.uint8).pin_memory() for g in job.dst}
            dist.barrier()
            job.sync_host(hs, hd)
            torch.cuda.synchronize()
            dist.barrier()
            for g in job.dst:
                assert np.array_equal(hd[g].numpy(), want[g]), f"random case {i} {cfg}: sync_host rank {g}"
        job.close()
        ran += 1
    assert ran >= n // 2, f"only {ran} random cases ran"


def full_case(runner, world, name):
    """Every byte of every generator buffer of a full-size config at `world`
    GPUs (tests/harness.py streamed compare): each process fills its own
    trainer ranks at the oracle's offsets; generator params are dealt out
    round-robin to the processes, each of which runs the oracle for its params
    and compares ALL generator ranks' bytes of them (peer buffers read through
    their IPC mappings); write coverage is summed over processes."""
    from paper_2505_24034_b200.runner import _wrap_device_ptr
    spec = runner.spec_for(name, world)
    # bounded host time: the whole 8B model; 4 decoder layers (+ embed / lm_head)
    # of 70B and 2 of the 405B slice -- same shapes per layer, same kernels
    layers = {"llama3-70b": 4, "llama3-405b-slice16": 2}.get(spec.cfg.model)
    if layers is not None:
        spec = runner.JobSpec(spec.cfg, world, n_layers=max(layers, spec.cfg.pp_train, spec.cfg.pp_gen))
    job = runner.SyncJob(spec, seed=0, fill=False)
    cfg = job.cfg
    ol = oracle.Layout(job.model, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                       cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    harness.fill_src_device(ol, 0, job.src)
    dev = torch.device("cuda", job.device)
    s_a, s_b = 0xA5, 0x5A
    counts = []
    for s in (s_b, s_a):
        for t in job.dst.values():
            t.fill_(s)
        torch.cuda.synchronize()
        dist.barrier()
        job.sync()
        torch.cuda.synchronize()
        dist.barrier()
        if s == s_b:
            counts = {q: harness.count_equal(t, s_b) for q, t in job.dst.items()}
    every = {q: job.dst[q] if q in job.dst else _wrap_device_ptr(job.dst_ptrs[q], job.D.rank_bytes(q), dev)
             for q in range(job.D.n_ranks)}
    mine = [gp for gp in range(ol.n_dst_params) if gp % world == dist.get_rank()]
    workers = max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", world)))
    n_eq_b = harness.streamed_compare(ol, 0, every, s_a, count_sentinel=s_b, workers=workers, gps=mine)
    tot = torch.tensor([n_eq_b[q] for q in range(job.D.n_ranks)], dtype=torch.int64, device=dev)
    dist.all_reduce(tot)
    for q, c in counts.items():
        pad = harness.dst_partition(ol, q)[1]
        assert c == int(tot[q]) + pad, f"{name}: generator rank {q}: {c - int(tot[q]) - pad} byte(s) not written"
    dist.barrier()
    job.close()


def rank0():
    return dist.get_rank() == 0


def main():
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_24034_b200 import runner
    if "--mc-only" in sys.argv:
        # NVLS multicast fan-out alone (run with LLRL_MC_UNICAST_PERIOD set: the
        # opt-in unicast egress split, fixed per process)
        toy_case(runner, world, world, 1, 1, "f32", "bf16", "colocated", dp=world, multicast=True)
        toy_case(runner, world, 3, 1, 2, "bf16", "bf16", "colocated", dp=world // 2 if world >= 4 else 2,
                 multicast=True)
        toy_case(runner, world, 2, 1, 1, "bf16", "bf16", "colocated", dp=world, multicast=True)
        dist.barrier()
        if dist.get_rank() == 0:
            print("MP_OK", flush=True)
        dist.destroy_process_group()
        return
    cases = [
        (2, 1, 2, "f32", "bf16", "disjoint"),
        (4, 1, 4, "f32", "bf16", "disjoint"),
        (8, 1, 8, "bf16", "bf16", "colocated"),
        (2, 4, 8, "bf16", "bf16", "colocated"),
        (1, 8, 8, "bf16", "fp8", "colocated"),
        (1, 8, 8, "bf16", "fp8", "rotated"),
        (3, 1, 4, "f32", "fp8", "colocated"),     # pull (multi-source) fp8 blocks across GPUs
        (2, 2, 8, "bf16", "fp8", "rotated"),
        (3, 2, 4, "f32", "f32", "disjoint"),
        (2, 2, 8, "bf16", "mxfp8", "rotated"),
        (2, 2, 8, "f32", "mxfp4", "colocated"),
        (2, 2, 8, "bf16", "nvfp4", "colocated"),     # per-tensor amax reduced across GPUs
        (4, 1, 2, "f32", "nvfp4", "disjoint"),
    ]
    # toy syncs are tiny (the product picks the register cast kernel for them):
    # run them through the TMA kernel of the large syncs as well
    for path in ("default", "6"):
        if path == "default":
            os.environ.pop("LLRL_CAST_VARIANT", None)
        else:
            os.environ["LLRL_CAST_VARIANT"] = path
        for c in cases:
            toy_case(runner, world, *c)
            if dist.get_rank() == 0:
                print("ok", path, c, flush=True)
        random_cases(runner, world, n=12 if path == "6" else 24, seed=2505 if path == "default" else 77)
    os.environ.pop("LLRL_CAST_VARIANT", None)
    toy_case(runner, world, 4, 1, 1, "f32", "bf16", "disjoint", dp=4)      # generator DP replicas
    toy_case(runner, world, 2, 2, 2, "bf16", "fp8", "disjoint", dp=2)
    toy_case(runner, world, 2, 2, 8, "bf16", "bf16", "colocated", ppt=2)       # pipeline re-staging
    toy_case(runner, world, 3, 1, 2, "f32", "mxfp8", "disjoint", ppt=2, ppg=2, dp=2)
    # NVLS multicast fan-out to DP replicas on different GPUs (NEXT f1)
    toy_case(runner, world, world, 1, 1, "f32", "bf16", "colocated", dp=world, multicast=True)
    toy_case(runner, world, 3, 1, 2, "bf16", "bf16", "colocated", dp=world // 2 if world >= 4 else 2,
             multicast=True)
    double_buffer_case(runner, world, 2, 1, 2, "f32", "bf16", "disjoint")   # f3 double buffering
    double_buffer_case(runner, world, 2, 2, 8, "bf16", "fp8", "rotated")
    nccl_replica_case(runner, world, 2, 1, 1, "f32", "bf16", world)       # a5 NCCL replication
    nccl_replica_case(runner, world, 2, 2, 2, "bf16", "fp8", world)
    nccl_replica_case(runner, world, world, 1, 1, "bf16", "bf16", world, mode=2)   # a5 all-gather
    nccl_replica_case(runner, world, world, 1, 1, "f32", "f32", world, mode=2)
    if rank0():
        print("ok nccl replicas", flush=True)
    if "--full" in sys.argv:
        for name in ("c2", "c3", "c4", "c5", "c7", "c8", "c10", "c11", "c12"):
            full_case(runner, world, name)
            if dist.get_rank() == 0:
                print("ok full", name, flush=True)
    dist.barrier()
    if dist.get_rank() == 0:
        print("MP_OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
