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
        # a5 (LLRL_PLAN_NCCL): every rank derives the same NCCL operations from the
        # plan (a collective must be entered identically everywhere), and the
        # replicated bytes match the layouts
        from synth import LayoutConfig
        for cfg in (LayoutConfig("b", "llama3-8b", 2, 1, 1, "bf16", "bf16", "disjoint", dp_gen=world),
                    LayoutConfig("b", "toy", 3, 1, 2, "f32", "bf16", "disjoint", dp_gen=world),
                    LayoutConfig("g", "llama3-8b", world, 1, 1, "bf16", "bf16", "colocated", dp_gen=world),
                    LayoutConfig("g", "toy", world, 1, 1, "f32", "f32", "colocated", dp_gen=world)):
            m = MODELS[cfg.model]
            S, D = llrl.describe(m, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, False,
                                 cfg.dp_gen)
            sd = [r * world // cfg.n_src for r in range(cfg.n_src)] if cfg.placement == "colocated" else [0] * cfg.n_src
            ns = D.n_ranks // cfg.dp_gen
            dd = ([q % world for q in range(D.n_ranks)] if cfg.placement == "colocated" else
                  [(q // ns) % world for q in range(D.n_ranks)])
            plan = llrl.Plan(S, D, sd, dd, nccl=True)
            infos = [(i.mode, i.n_broadcasts, i.n_allgathers, i.bytes)
                     for i in (plan.nccl_info(d) for d in range(plan.stats().n_devices))]
            allinfo = [None] * world
            dist.all_gather_object(allinfo, infos)
            assert all(a == infos for a in allinfo), "ranks derived different NCCL operations"
            if cfg.name == "g":                  # FSDP chunks all-gathered: no kernel work at all
                assert all(i[0] == 2 for i in infos) and plan.stats().n_items == 0
                data = sum(D.param_view(0, gp).rows * D.param_view(0, gp).cols for gp in range(D.n_params))
                es = 4 if cfg.src_dtype == "f32" else 2
                assert all(i[3] == data * es * (world - 1) // world for i in infos)
            else:                                # replicas 1.. by broadcast of replica 0's buffer
                assert all(i[0] == 1 for i in infos)
                for d, i in enumerate(infos):
                    reps = [q for q in range(ns, D.n_ranks) if dd[q] == d]
                    assert i[3] == sum(D.rank_bytes(q) for q in reps)
                    assert i[1] == len({q % ns for q in range(D.n_ranks) if dd[q] == d})
                # the kernels write replica 0 only
                runs = plan.runs()
                assert runs.size and int(runs["dst_rank"].max()) < ns
        # runner._exchange_fds (multicast egress split: every process maps its peers'
        # replica memory): all-to-all fd passing over Unix sockets, checked with pipes
        pipes = [os.pipe() for _ in range(2)]
        got = runner._exchange_fds(f"llrl-test-{port}", rank, world, [w for _, w in pipes])
        assert sorted(got) == [p for p in range(world) if p != rank] and all(len(v) == 2 for v in got.values())
        for p, fds in got.items():
            for k, fd in enumerate(fds):
                os.write(fd, f"{rank}>{p}:{k};".encode())
                os.close(fd)
        dist.barrier()
        for k, (r, _) in enumerate(pipes):
            data = os.read(r, 4096).decode()
            os.close(r)
            want = sorted(f"{s}>{rank}:{k}" for s in range(world) if s != rank)
            assert sorted(x for x in data.split(";") if x) == want, data
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
