"""Torch plumbing around libllrl: device buffers, streams, process groups and
the IPC exchange that maps peer buffers for the push kernels.

One process per GPU (torch.distributed, one rank per device on one node), or a
single process driving device 0 when every logical trainer/generator rank is
placed on one GPU.  Every byte of the sync itself is moved by libllrl's
kernels; this module only allocates, maps and calls.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from . import llrl
from synth import MODELS, CONFIGS, LayoutConfig, placement


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


@dataclass
class JobSpec:
    cfg: LayoutConfig
    n_gpus: int
    n_layers: int | None = None       # override (e.g. a layer slice that fits one GPU)
    with_embed: int | None = None

    def model(self):
        m = MODELS[self.cfg.model]
        kw = {}
        if self.n_layers is not None:
            kw["n_layers"] = self.n_layers
        if self.with_embed is not None:
            kw["with_embed"] = self.with_embed
        return m.replace(**kw) if kw else m


class SyncJob:
    """One trainer->generator layout pair placed on `n_gpus` GPUs.

    In a torch.distributed job the calling process owns device ``rank``; without
    one, the job must fit one device (n_gpus == 1)."""

    def __init__(self, spec: JobSpec, device: int | None = None, seed: int = 0, fill: bool = True,
                 multicast: bool = False, replicate: str = "push", double_buffer: bool = False):
        self.spec = spec
        self.cfg = cfg = spec.cfg
        self.model = spec.model()
        d = _dist()
        self.world = d.get_world_size() if d else 1
        self.rank = d.get_rank() if d else 0
        if self.world > 1:
            assert self.world == spec.n_gpus, "one process per GPU"
        else:
            assert spec.n_gpus == 1, "multi-GPU jobs run one process per GPU (torchrun)"
        self.device = self.rank if device is None else device
        torch.cuda.set_device(self.device)
        self.S, self.D = llrl.describe(self.model, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype,
                                       cfg.dst_dtype, cfg.fsdp_inner, cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
        self.src_dev, self.dst_dev = placement(cfg, spec.n_gpus)
        # plain replication.  "push" (and multicast) write every
        # generator replica from the trainer shards in the fused kernels; "nccl" makes
        # an LLRL_PLAN_NCCL plan: the library replaces replica copies by ncclBroadcast
        # or the whole sync by ncclAllGathers where the mapping is a plain
        # replication (DESIGN R17, R18), all inside llrl_sync.
        if replicate not in ("push", "nccl"):
            raise ValueError(f"replicate must be 'push' or 'nccl', not {replicate!r}")
        if replicate == "nccl" and multicast:
            raise ValueError("replicate='nccl' and multicast are exclusive")
        self.replicate = replicate
        self.plan = llrl.Plan(self.S, self.D, self.src_dev, self.dst_dev, multicast=multicast,
                              nccl=replicate == "nccl")
        dev = torch.device("cuda", self.device)
        self.src = {r: torch.empty(self.S.rank_bytes(r), dtype=torch.uint8, device=dev)
                    for r in range(self.S.n_ranks) if self.src_dev[r] == self.device}
        self._mc = []
        self.mc_ranks = set()
        self._mc_peer_ptrs = {}
        self.dst = {}
        if multicast and self.world > 1:
            self._setup_multicast()
        for g in range(self.D.n_ranks):
            if self.dst_dev[g] == self.device and g not in self.dst:
                self.dst[g] = torch.empty(self.D.rank_bytes(g), dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.current_stream(dev)
        if fill:
            self.fill(seed)
        self.comm = None
        self._opened = []
        self.src_ptrs = [self.src[r].data_ptr() if r in self.src else 0 for r in range(self.S.n_ranks)]
        self.dst_ptrs = [self.dst[g].data_ptr() if g in self.dst else self._mc_peer_ptrs.get(g, 0)
                         for g in range(self.D.n_ranks)]
        # NEXT f3: double-buffered generator weights.  `dst` is what the next sync
        # writes, `front` what the generator reads; swap() exchanges them once a
        # sync completed, so generation continues during the sync.
        self.double_buffer = double_buffer
        self._sets = None
        self.front = self.dst
        if double_buffer:
            if multicast:
                raise ValueError("double_buffer with multicast is not supported")
            other = {g: torch.empty_like(t) for g, t in self.dst.items()}
            optrs = [other[g].data_ptr() if g in other else 0 for g in range(self.D.n_ranks)]
            self._sets = [(self.dst, self.dst_ptrs), (other, optrs)]
            self.front = other
        if self.world > 1:
            self._exchange()
            if self.plan.nccl_info(0).mode:       # llrl_nccl_attach: collective over every process
                holder = [llrl.nccl_unique_id() if self.rank == 0 else None]
                _dist().broadcast_object_list(holder, src=0)
                self.plan.nccl_attach(self.device, holder[0], self.rank, self.world)
        elif cfg.dst_dtype == "nvfp4":
            self.comm = llrl.Comm(self.device)     # NVFP4 keeps its amax table in the comm buffer

    # -- setup ---------------------------------------------------------------
    def fill(self, seed: int):
        for r, t in self.src.items():
            llrl.fill_synthetic(self.S, r, t.data_ptr(), seed, self.stream.cuda_stream)
        torch.cuda.synchronize(self.device)

    def _exchange(self):
        """Map every peer's rank buffers and completion flags (cudaIpc over NVLink)."""
        dist = _dist()
        self.comm = llrl.Comm(self.device)
        mine = exchange_meta(self.device, self.comm.export(),
                             {r: llrl.ipc_handle(t.data_ptr()) for r, t in self.src.items()},
                             {g: llrl.ipc_handle(t.data_ptr()) for g, t in self.dst.items()
                              if g not in self.mc_ranks})   # multicast buffers are reached via the MC VA
        extra = None
        if self._sets is not None:
            mine["dst1"] = {g: llrl.ipc_handle(t.data_ptr()) for g, t in self._sets[1][0].items()}
            extra = {"dst1": self._sets[1][1]}
        allm = [None] * self.world
        dist.all_gather_object(allm, mine)
        opened = {}

        def opener(handle):
            base = llrl.ipc_open(handle, 0)
            opened[handle] = base
            return base

        flags = map_peers(allm, self.device, self.src_ptrs, self.dst_ptrs, opener, extra)
        for dev, h in flags.items():
            self.comm.import_peer(dev, h)
        self._opened = [(b, 0) for b in opened.values()]
        dist.barrier()

    def mc_positions(self):
        """Generator rank positions whose DP replicas sit on pairwise different GPUs
        (the plan's multicast eligibility rule, R12 numbering q = d*NS + pos)."""
        dp = self.cfg.dp_gen
        ns = self.D.n_ranks // dp
        out = []
        for pos in range(ns):
            devs = [self.dst_dev[d * ns + pos] for d in range(dp)]
            if dp > 1 and len(set(devs)) == dp:
                out.append(pos)
        return out, ns

    def _setup_multicast(self):
        """NVLS multicast (NEXT f1): one multicast object per eligible position; rank 0
        creates them and passes the POSIX fds over a Unix socket (SCM_RIGHTS); every
        process joins with its GPU; replica GPUs use the bound memory as their
        generator buffer."""
        import socket
        dist = _dist()
        positions, ns = self.mc_positions()
        if not positions:
            return
        name = f"\0llrl-mc-{os.environ.get('MASTER_PORT', '0')}-{os.getuid()}-{id(self.plan) & 0xffff}"
        holder = [name]
        dist.broadcast_object_list(holder, src=0)
        name = holder[0]
        sizes, fds, bufs = [], [], []
        if self.rank == 0:
            for pos in positions:
                buf, fd = llrl.McBuf.create(self.world, self.D.rank_bytes(pos))
                bufs.append(buf)
                fds.append(fd)
                sizes.append(buf.size)
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(name)
            srv.listen(self.world)
            dist.broadcast_object_list([sizes], src=0)
            for _ in range(self.world - 1):
                conn, _ = srv.accept()
                socket.send_fds(conn, [b"llrl"], fds)
                conn.close()
            srv.close()
            for fd in fds:
                os.close(fd)
        else:
            holder = [None]
            dist.broadcast_object_list(holder, src=0)
            sizes = holder[0]
            conn = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            import time
            for _ in range(200):
                try:
                    conn.connect(name)
                    break
                except OSError:
                    time.sleep(0.05)
            _, fds, _, _ = socket.recv_fds(conn, 16, len(positions))
            conn.close()
            for fd, size in zip(fds, sizes):
                bufs.append(llrl.McBuf.import_fd(fd, self.world, size))
                os.close(fd)
        dst_mc = [0] * self.D.n_ranks
        dev = torch.device("cuda", self.device)
        for pos, buf in zip(positions, bufs):
            local, mcva = buf.join(self.device)           # blocks until every GPU joined
            for d in range(self.cfg.dp_gen):
                q = d * ns + pos
                dst_mc[q] = mcva
                if self.dst_dev[q] == self.device:
                    self.dst[q] = _wrap_device_ptr(local, self.D.rank_bytes(q), dev)
                    self.mc_ranks.add(q)
            self.mc_ranks.update(d * ns + pos for d in range(self.cfg.dp_gen))
        self._mc = bufs
        self.plan.set_multicast(self.device, dst_mc)
        dist.barrier()
        # egress split (plan.cpp: a share of each position's items is pushed to every
        # replica as plain peer stores): map the peers' replica memory here
        peer_fds = _exchange_fds(name + "-x", self.rank, self.world, [b.export_local() for b in bufs])
        for k, (pos, buf) in enumerate(zip(positions, bufs)):
            for d in range(self.cfg.dp_gen):
                q = d * ns + pos
                if self.dst_dev[q] != self.device:
                    self._mc_peer_ptrs[q] = buf.map_peer(peer_fds[self.dst_dev[q]][k], self.device)
        for fds in peer_fds.values():
            for fd in fds:
                os.close(fd)
        dist.barrier()

    def swap(self):
        """Double buffering (f3): make the buffers the last sync wrote the generator's
        front and target the other set with the next sync.  Every process swaps
        after the same sync (peer pointer sets stay paired); order it after the
        sync's completion on the generator's stream (the sync's stream, or an
        event recorded on it)."""
        if self._sets is None:
            raise ValueError("swap() needs SyncJob(double_buffer=True)")
        k = 1 if self.dst is self._sets[0][0] else 0
        self.front = self.dst
        self.dst, self.dst_ptrs = self._sets[k]

    # -- the hot path ----------------------------------------------------------
    def sync(self, stream=None):
        s = stream if stream is not None else self.stream
        if self._in_plan():              # a GPU without trainer or generator ranks has no work
            self.plan.sync(self.comm, self.device, self.src_ptrs, self.dst_ptrs, s.cuda_stream)

    def sync_nv_amax(self, amax, stream=None):
        """llrl_sync_nv_amax: an NVFP4 sync in one pass with the caller's per-tensor
        amax (a float32 CUDA tensor on this device, one value per plan tensor id)."""
        s = stream if stream is not None else self.stream
        assert amax.dtype == torch.float32 and amax.is_cuda and amax.numel() >= self.plan.nv_num_tensors()
        if self._in_plan():
            self.plan.sync_nv_amax(self.comm, self.device, amax.data_ptr(), self.src_ptrs, self.dst_ptrs,
                                   s.cuda_stream)

    def sync_group(self, group, stream=None):
        s = stream if stream is not None else self.stream
        if self._in_plan():
            self.plan.sync_group(self.comm, self.device, group, self.src_ptrs, self.dst_ptrs, s.cuda_stream)

    def src_group_views(self, group):
        """Views of this device's trainer bytes of one layer group (for an optimizer step)."""
        dt = torch.float32 if self.cfg.src_dtype == "f32" else torch.bfloat16
        out = []
        for r, t in self.src.items():
            lo, hi = self.plan.group_range(0, r, group)
            if lo >= 0:
                out.append(t[lo:hi].view(dt))
        return out

    def overlapped_step(self, opt_fn, opt_stream, stream=None):
        """NEXT f3: per layer group, the optimizer (opt_fn(views) on opt_stream)
        updates group g while llrl_sync_group streams group g-1 out: the sync of a
        layer starts as soon as that layer's update is done."""
        s = stream if stream is not None else self.stream
        if self.world > 1 and self.plan.stats().n_fp8_pull_blocks:
            # multi-source fp8 blocks are PULLED from peers' trainer buffers: group g's
            # pull would only be ordered after the LOCAL optimizer event, so a peer's
            # half-updated (or next-step) weights could be read.  Refused rather than
            # racing; llrl_sync_host orders pulls with "staged" handshakes instead.
            raise ValueError("overlapped_step: the plan pulls fp8 blocks from peer GPUs (uneven FSDP chunks); "
                             "use sync() after the optimizer step, or sync_host")
        n = self.plan.num_groups()
        opt_stream.wait_stream(s)
        for g in range(n):
            with torch.cuda.stream(opt_stream):
                opt_fn(self.src_group_views(g))
                ev = torch.cuda.Event()
                ev.record(opt_stream)
            s.wait_event(ev)
            self.sync_group(g, s)

    def sync_host(self, host_src, host_dst, stream=None):
        """End-to-end entry: host trainer shards in, host generator shards out."""
        s = stream if stream is not None else self.stream
        hs = [host_src[r].data_ptr() if r in host_src else 0 for r in range(self.S.n_ranks)]
        hd = [host_dst[g].data_ptr() if g in host_dst else 0 for g in range(self.D.n_ranks)]
        if self._in_plan():
            self.plan.sync_host(self.comm, self.device, hs, hd, self.src_ptrs, self.dst_ptrs, s.cuda_stream)

    def _in_plan(self):
        return self.device in set(self.plan.src_device) | set(self.plan.dst_device)

    def num_launches(self):
        return self.plan.num_launches(self.device) if self._in_plan() else 0

    def close(self):
        for p, off in self._opened:
            try:
                llrl.ipc_close(p, off)
            except llrl.LlrlError:
                pass
        self._opened = []
        if self.comm is not None:
            self.comm.close()
            self.comm = None
        self.plan.close()
        self.dst = {}
        self.front = {}
        self._sets = None
        for b in self._mc:
            b.close()
        self._mc = []


class _CudaArray:
    """Minimal __cuda_array_interface__ holder: a torch view of library-owned memory."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": (nbytes,), "typestr": "|u1", "version": 3}


def _wrap_device_ptr(ptr, nbytes, device):
    return torch.as_tensor(_CudaArray(ptr, nbytes), device=device)


def exchange_meta(device, flag_handle, src_handles, dst_handles):
    """What one process publishes: its device, its flag-buffer IPC handle and, per
    owned rank buffer, (allocation IPC handle, byte offset in the allocation)."""
    return {"dev": device, "flag": flag_handle, "src": dict(src_handles), "dst": dict(dst_handles)}


def map_peers(all_meta, my_device, src_ptrs, dst_ptrs, opener, extra=None):
    """Fill src_ptrs / dst_ptrs (in place) with peer-mapped addresses of every rank
    buffer other processes own.  Each distinct allocation handle is opened once
    (several rank buffers may share one caching-allocator segment); returns
    {peer device: flag handle}.  Pure host logic (tested on gloo, CPU)."""
    bases = {}
    flags = {}
    for m in all_meta:
        if m["dev"] == my_device:
            continue
        flags[m["dev"]] = m["flag"]
        tables = [("src", src_ptrs), ("dst", dst_ptrs)] + list((extra or {}).items())
        for table, ptrs in tables:
            for r, (h, off) in m[table].items():
                if h not in bases:
                    bases[h] = opener(h)
                ptrs[int(r)] = bases[h] + off
    return flags


def _exchange_fds(tag, rank, world, fds):
    """All-to-all exchange of POSIX fds between the processes of one node (one
    abstract Unix socket per process, SCM_RIGHTS); process rank == GPU ordinal.
    Returns {peer rank: [its fds, in order]}; closes the fds sent."""
    import socket
    import threading
    import time
    dist = _dist()

    def sock_name(r):
        return f"\0{tag}-{r}"
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(sock_name(rank))
    srv.listen(world)
    dist.barrier()
    got = {}

    def acceptor():
        for _ in range(world - 1):
            conn, _ = srv.accept()
            msg, rfds, _, _ = socket.recv_fds(conn, 64, max(1, len(fds)))
            got[int(msg.decode())] = list(rfds)
            conn.close()
    th = threading.Thread(target=acceptor, daemon=True)
    th.start()
    for p in range(world):
        if p == rank:
            continue
        c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        for _ in range(400):
            try:
                c.connect(sock_name(p))
                break
            except OSError:
                time.sleep(0.05)
        socket.send_fds(c, [str(rank).encode()], fds)
        c.close()
    th.join(timeout=120)
    srv.close()
    for fd in fds:
        os.close(fd)
    return got


def spec_for(name: str, n_gpus: int) -> JobSpec:
    """The benchmark job of config `name` at `n_gpus` (SURVEY.md §8(d) placements).

    70B at G=1 does not fit one B200 (282 GB): a 40-layer slice with embed /
    lm_head is used, as SURVEY §8(d) specifies."""
    cfg = CONFIGS[name]
    if cfg.model == "llama3-70b" and n_gpus == 1:
        return JobSpec(cfg, n_gpus, n_layers=40)
    return JobSpec(cfg, n_gpus)


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
