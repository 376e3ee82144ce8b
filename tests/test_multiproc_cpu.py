"""N>1 host logic on CPU with world_size-2, -4 and -8 gloo process groups: every rank
builds the same plan independently, the per-device shares add up to the whole
sync, each device's expected arrivals match the senders that signal it, and
the IPC exchange (runner.map_peers) maps every peer buffer a device's work
touches, opening each allocation once."""
from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2505_24034_b200 import llrl, runner
        from synth import CONFIGS, MODELS, placement
        for name in ("c2", "c3", "c5"):
            cfg = CONFIGS[name]
            S, D = llrl.describe(MODELS[cfg.model], cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype,
                                 cfg.dst_dtype, cfg.fsdp_inner)
            sd, dd = placement(cfg, world)
            plan = llrl.Plan(S, D, sd, dd)
            mine = plan.device_bytes(rank)
            info = plan.device_info(rank)
            allb = [None] * world
            dist.all_gather_object(allb, (mine, plan.traffic(), info.n_signal, info.n_senders_in))
            tr = allb[0][1]
            assert all(a[1] == tr for a in allb), "ranks built different plans"
            st = plan.stats()
            assert sum(a[0]["hbm_read"] for a in allb) == st.src_bytes
            assert sum(a[0]["hbm_write"] for a in allb) == st.dst_bytes
            assert sum(a[0]["nvl_tx"] for a in allb) == sum(a[0]["nvl_rx"] for a in allb)
            for d in range(world):   # push plans: who signals whom == off-diagonal traffic
                assert allb[d][2] == sum(1 for x in range(world) if x != d and tr[d][x] > 0)
                assert allb[d][3] == sum(1 for s in range(world) if s != d and tr[s][d] > 0)
            # IPC exchange logic with fake handles: one allocation per process holding all its ranks
            own_src = {r: (f"h{rank}".encode(), 1000 * r) for r in range(S.n_ranks) if sd[r] == rank}
            own_dst = {g: (f"h{rank}".encode(), 5000 + 1000 * g) for g in range(D.n_ranks) if dd[g] == rank}
            meta = runner.exchange_meta(rank, f"f{rank}".encode(), own_src, own_dst)
            allm = [None] * world
            dist.all_gather_object(allm, meta)
            src_ptrs = [0] * S.n_ranks
            dst_ptrs = [0] * D.n_ranks
            for r in own_src:
                src_ptrs[r] = 1
            for g in own_dst:
                dst_ptrs[g] = 1
            opened = []

            def opener(h):
                opened.append(h)
                return 10 ** 9 * (int(h.decode()[1:]) + 1)

            for m in allm:                       # a second generator set (double buffering, f3)
                m["dst1"] = {g: (h, off + 500) for g, (h, off) in m["dst"].items()}
            dst1 = [0] * D.n_ranks
            flags = runner.map_peers(allm, rank, src_ptrs, dst_ptrs, opener, {"dst1": dst1})
            assert sorted(opened) == sorted({f"h{p}".encode() for p in range(world) if p != rank})
            assert set(flags) == {p for p in range(world) if p != rank}
            assert all(src_ptrs) and all(dst_ptrs)
            for g in range(D.n_ranks):
                if dd[g] != rank:
                    assert dst_ptrs[g] == 10 ** 9 * (dd[g] + 1) + 5000 + 1000 * g
                    assert dst1[g] == dst_ptrs[g] + 500
        # a5 NCCL-style replica broadcast (runner.broadcast_plan / run_broadcasts) on gloo:
        # replica 0's buffers reach every replica, other ranks' buffers stay untouched
        import torch
        for dp, ns in ((world, 1), (world, 2), (2, 3)):
            n = dp * ns
            dd = [(d + pos) % world if dp == world else (pos + d * (world // 2)) % world
                  for d in range(dp) for pos in range(ns)]
            bp = runner.broadcast_plan(dd, dp)
            assert [b[0] for b in bp] == list(range(ns))
            assert all(b[1] == dd[b[0]] and len(b[2]) == dp for b in bp)
            groups = runner.make_broadcast_groups(dist, bp)
            bufs = {qq: torch.full((64,), -1.0) for qq in range(n) if dd[qq] == rank}
            for qq in bufs:
                if qq < ns:                       # replica 0 holds the synced bytes
                    bufs[qq] = torch.arange(64, dtype=torch.float32) + 100 * qq
            runner.run_broadcasts(dist, groups, rank, bufs)
            for qq, t in bufs.items():
                assert torch.equal(t, torch.arange(64, dtype=torch.float32) + 100 * (qq % ns)), (dp, ns, qq)
        with pytest.raises(ValueError):
            runner.broadcast_plan([0, 0], 2)      # replicas of one position on one GPU
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multiprocess_plan_and_exchange_gloo(world):
    from paper_2505_24034_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
