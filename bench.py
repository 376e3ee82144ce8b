#!/usr/bin/env python
"""bench.py -- DDMA trainer->generator weight-sync latency on B200 (LlamaRL,
arxiv 2505.24034 §5.2; BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W --config c2]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
  python bench.py --impl reference ...      # the CPU oracle on host cores

A step is one whole sync of the configuration's
full model: every trainer shard read, every generator shard written.  At N=1
the workload is configs[1] (C2, Llama-3.1 8B fp32 FSDP=4 -> bf16 TP=4, all
logical ranks on GPU 0); at N>1 the same model with trainer ranks on GPUs
[0, N/2) and generator ranks on [N/2, N), i.e. strong scaling.
Inputs (GBs) are larger than the 126 MB L2, so no flush is needed between
steps.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "weight-sync latency (ms) and NVLink GB/s/GPU for Llama-3 8B/70B at 1/2/4/8 B200"
NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction (900 nominal)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, gpus):
        self.gpus = gpus
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                      "-i", ",".join(map(str, self.gpus))], capture_output=True, text=True,
                                     timeout=5).stdout
                for line in out.strip().splitlines():
                    f = [x.strip() for x in line.split(",")]
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        load = [s for s in self.samples if num(s[-1]) and num(s[-1]) > 0] or self.samples
        sm = sorted(num(s[1]) for s in load if num(s[1]) is not None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in load for n, v in zip(names, s[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": num(load[0][2]), "reasons": reasons,
                "samples": len(load)}


def _dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _allmax(x):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _allsum(x):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def _barrier():
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()


# ---------------------------------------------------------------- CPU oracle legs
#
# SURVEY §8(d) "How to time the oracle": the oracle (oracle/oracle.c, as it
# stands) on host copies of the trainer shards of the WHOLE workload, timed
# single-threaded and parameter-parallel (one generator parameter per task,
# nproc threads: the "std::thread x nproc" leg; ctypes releases the GIL), with
# nproc and the lscpu model stated.  The inputs are generated on the host by
# synth.fast (the input generator) at the oracle's offsets -- nothing of the
# product is loaded on these legs.


def _model_for(cfg, n_gpus):
    """The workload's model: runner.spec_for's rule (70B at G=1 is the 40-layer
    slice with embed / lm_head), without importing the product."""
    from synth import MODELS
    m = MODELS[cfg.model]
    return m.replace(n_layers=40) if cfg.model == "llama3-70b" and n_gpus == 1 else m


def _cpu_model_name():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class OracleWorkload:
    """Host trainer buffers of the whole workload + reusable generator buffers."""

    def __init__(self, cfg, n_gpus, seed=0):
        import numpy as np
        import oracle
        from synth import fast
        self.model = _model_for(cfg, n_gpus)
        ol = oracle.Layout(self.model, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype,
                           cfg.fsdp_inner, cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
        assert ol.status == 0, ol.status
        self.ol = ol
        es = 4 if cfg.src_dtype == "f32" else 2
        self.src = []
        for r in range(ol.n_src):
            buf = np.zeros(ol.src_rank_bytes(r), np.uint8)
            for p in range(ol.n_src_params):
                off, r0, r1, c0, c1 = ol.src_piece(r, p)
                if r1 > r0 and c1 > c0:
                    n = (r1 - r0) * (c1 - c0) * es
                    fast.fill(buf[off:off + n], seed, p, ol.src_param_info(p)[2] == 2, cfg.src_dtype, r0, r1, c0, c1)
            self.src.append(buf)
        self.dst = [np.zeros(ol.dst_rank_bytes(q), np.uint8) for q in range(ol.n_dst)]
        self.saddr = [b.ctypes.data for b in self.src]
        self.daddr = [b.ctypes.data for b in self.dst]
        # biggest generator params first so the thread pool's tail is short
        size = [sum(ol.dst_param(q, gp)[0] * ol.dst_param(q, gp)[1] for q in range(min(ol.n_dst, 1)))
                for gp in range(ol.n_dst_params)]
        self.order = sorted(range(ol.n_dst_params), key=lambda gp: -size[gp])
        self.elements = sum(ol.src_param_info(p)[0] * ol.src_param_info(p)[1] for p in range(ol.n_src_params))

    def run(self, threads):
        """One whole sync by the oracle; returns wall seconds."""
        import concurrent.futures as cf
        ol = self.ol
        t0 = time.perf_counter()
        if threads <= 1:
            rc = ol.sync_addrs(self.saddr, self.daddr, (0, ol.n_dst_params))
            assert rc == 0, rc
        else:
            with cf.ThreadPoolExecutor(threads) as ex:
                rcs = list(ex.map(lambda gp: ol.sync_addrs(self.saddr, self.daddr, (gp, gp + 1)), self.order))
            assert all(rc == 0 for rc in rcs), rcs
        return time.perf_counter() - t0


def cpu_baseline(cfg, n_gpus, single_thread=True):
    """The oracle on the whole workload: parameter-parallel over nproc threads (the
    reported value), and single-threaded (also the whole workload)."""
    nproc = os.cpu_count() or 1
    t0 = time.perf_counter()
    w = OracleWorkload(cfg, n_gpus)
    t_gen = time.perf_counter() - t0
    par = w.run(nproc)
    out = {"value": round(par * 1e3, 1), "unit": "ms", "cores": nproc, "kind": "oracle",
           "sample": f"the whole workload ({w.model.n_layers} layers + embed/lm_head of {cfg.model}, "
                     f"{w.elements / 1e9:.3f} G trainer elements), no extrapolation: oracle/oracle.c "
                     f"parameter-parallel (one generator parameter per task) on {nproc} threads; host "
                     f"{_cpu_model_name()}, nproc {nproc}; inputs generated on the host by synth.fast at the "
                     f"oracle's offsets ({t_gen:.1f} s, not timed)",
           "cpu_model": _cpu_model_name(), "nproc": nproc, "parallel_ms": round(par * 1e3, 1)}
    if single_thread:
        st = w.run(1)
        out["single_thread_ms"] = round(st * 1e3, 1)
        out["parallel_speedup"] = round(st / par, 2)
    return out


def run_reference(args):
    """--impl reference: the CPU oracle as it stands on the host cores (rank 0
    only): every step one whole sync of the workload, parameter-parallel over
    nproc threads -- no sample, no extrapolation."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    nproc = os.cpu_count() or 1
    w = OracleWorkload(cfg, args.gpus)
    for _ in range(args.warmup):
        w.run(nproc)
    ts = [w.run(nproc) for _ in range(args.steps)]
    step_ms = sum(ts) / len(ts) * 1e3
    sample = (f"every step the whole workload ({w.model.n_layers} layers + embed/lm_head of {cfg.model}, "
              f"{w.elements / 1e9:.3f} G trainer elements): oracle/oracle.c parameter-parallel on {nproc} threads "
              f"(host {_cpu_model_name()}); no extrapolation")
    line = {"impl": "reference", "metric": METRIC, "value": round(step_ms, 3), "unit": "ms",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "ms_min": round(min(ts) * 1e3, 3), "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": f"{cfg.src_dtype}->{cfg.dst_dtype}", "data": DATA, "config": config_dict(cfg, args, w.model),
            "cpu_baseline": {"value": round(step_ms, 3), "unit": "ms", "cores": nproc, "kind": "oracle",
                             "sample": sample, "cpu_model": _cpu_model_name(), "nproc": nproc},
            "e2e": {"value": round(step_ms, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


DATA = "synthetic (counter-based Llama-init-scale weights)"


def _workload_name(cfg, n):
    return f"{cfg.name}: {cfg.notes} @ {n} GPU(s)"


def _small_working_set(cfg, model, n_gpus):
    """Syncs whose per-GPU bytes could stay in the 126 MB L2 are timed one at a time
    with L2 flushed before each (timing rule); decided from the layouts only, so
    both arms report the same config."""
    import oracle
    ol = oracle.Layout(model, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                       cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    tot = sum(ol.src_rank_bytes(r) for r in range(ol.n_src)) + sum(ol.dst_rank_bytes(q) for q in range(ol.n_dst))
    return tot / n_gpus < (1 << 30)


def config_dict(cfg, args, model):
    """The `config` object of both arms' JSON lines (identical for one invocation)."""
    small = _small_working_set(cfg, model, args.gpus)
    return {"workload": _workload_name(cfg, args.gpus), "shapes": cfg.model,
            "dp_gen": cfg.dp_gen, "pp_train": cfg.pp_train, "pp_gen": cfg.pp_gen,
            "max_ctas": args.max_ctas or "all SMs", "multicast": bool(args.multicast),
            "replicate": args.replicate,
            "timing": "isolated syncs (barrier before each)" if (args.step_sync or small) else "back-to-back syncs",
            "regime": ("all ranks on one GPU: local HBM re-layout + cast" if args.gpus == 1 else
                       f"{cfg.placement} placement over {args.gpus} GPUs: fused pushes over NVLink"
                       " (G=1 and G>=2 are different regimes; compare each to roofline.t_lb_ms)"),
            "n_layers": model.n_layers, "fsdp": cfg.fsdp, "tp_train": cfg.tp_train,
            "tp_gen": cfg.tp_gen, "placement": args.placement or cfg.placement,
            "l2": ("working set < 1 GB: L2 flushed (512 MB write) before every timed sync, syncs "
                   "timed one at a time" if small else "inputs >> 126 MB L2 (no flush needed)")}


# ---------------------------------------------------------------- our arm

def run_llrl(args):
    import torch
    from paper_2505_24034_b200 import build
    build.build()
    from paper_2505_24034_b200 import runner
    world, rank, local = _dist_setup(args)
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    spec = runner.spec_for(args.config, args.gpus)
    if args.layers is not None:           # profiling only (ncu replay of a smaller model)
        spec = runner.JobSpec(spec.cfg, spec.n_gpus, n_layers=args.layers)
    if args.placement:
        import dataclasses
        spec = runner.JobSpec(dataclasses.replace(spec.cfg, placement=args.placement), spec.n_gpus, spec.n_layers)
    job = runner.SyncJob(spec, device=local, seed=0, multicast=args.multicast, replicate=args.replicate)
    if args.max_ctas:
        job.plan.set_max_ctas(job.device, args.max_ctas)
    cfg = job.cfg
    stream = job.stream

    # warm-up (also uploads the device tables)
    for _ in range(args.warmup):
        job.sync()
    _barrier()
    # working sets that could stay in the 126 MB L2 between syncs are measured one
    # sync at a time with L2 flushed before each (timing rule); larger ones stream
    small = _small_working_set(cfg, job.model, args.gpus)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=torch.device("cuda", local)) if small else None

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler([local]) as clk:
        time.sleep(0.25)       # let the sampler start before the timed region
        _barrier()
        if args.step_sync or small:
            # isolated syncs: every GPU idle and every rank past a barrier before each
            # one, so no sync overlaps the previous one's tail (single-sync latency);
            # small working sets: L2 flushed (a 512 MB write) before each sync
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for k in range(args.steps):
                torch.cuda.synchronize()
                _barrier()
                with torch.cuda.stream(stream):
                    if small:
                        # the flush (a 512 MB write, ~0.1 ms) also keeps the GPU busy while
                        # the host enqueues the sync, so the events time the GPU's work
                        # only, not the host's launch path
                        flush.fill_(k & 0xFF)
                    evs[k][0].record(stream)
                    job.sync()
                    evs[k][1].record(stream)
            torch.cuda.synchronize()
            _barrier()
        else:
            with torch.cuda.stream(stream):
                ev[0].record(stream)
                for k in range(args.steps):
                    job.sync()
                    ev[k + 1].record(stream)
        _barrier()
    floor_us = None
    if small:
        # context for the isolated-sync number: the same protocol (flush, event,
        # one kernel, event) around a one-byte torch kernel -- the launch + event
        # floor any single-kernel sync pays on this box
        fl = []
        for k in range(args.steps):
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                flush[:1].add_(1)
                b.record(stream)
            fl.append((a, b))
        torch.cuda.synchronize()
        floor_us = round(1000 * sorted(a.elapsed_time(b) for a, b in fl)[len(fl) // 2], 2)
    if args.step_sync or small:
        step_ms = [_allmax(a.elapsed_time(b)) for a, b in evs]
        ms = sum(step_ms) / len(step_ms)
        ms_min = min(step_ms)
    else:
        step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
        total_ms = ev[0].elapsed_time(ev[-1])
        ms = _allmax(total_ms / args.steps)
        ms_min = _allmax(min(step_ms))
    launches = int(_allsum(job.num_launches() * args.steps))

    # roofline: the binding resource of the binding GPU (the plan is identical on
    # every rank, so each rank can evaluate every device); achieved = its
    # algorithmic bytes per sync / the max-over-ranks device time per sync.
    hbm_peak, peak_src = _peaks()
    best = None
    ndev = job.plan.stats().n_devices           # < n_gpus when GPUs only take NCCL replicas
    for d in range(ndev):
        b = job.plan.device_bytes(d)
        for res, nbytes, peak in (("hbm", b["hbm_read"] + b["hbm_write"], hbm_peak),
                                  ("nvlink", max(b["nvl_tx"], b["nvl_rx"]), NVLINK_PEER_GBS)):
            t = nbytes / peak / 1e6
            if best is None or t > best[0]:
                best = (t, res, nbytes, peak, d)
    t_lb, res, nbytes, peak, bdev = best
    roof = {"bound": res, "achieved": round(nbytes / ms / 1e6, 1), "peak": peak, "unit": "GB/s",
            "peak_source": peak_src if res == "hbm" else "measured peer copy per direction (B200_PROFILING.md)"}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    nominal = 8000.0 if res == "hbm" else 900.0                      # B200 HBM3e / NVLink 5 per direction
    roof["frac_nominal"] = round(roof["achieved"] / nominal, 4)
    roof["nominal_peak"] = nominal
    roof["traffic"] = _ncu_traffic(args.config, args.gpus)
    info = job.plan.device_info(bdev)
    kern = []
    if info.n_cast_items:
        kern.append("llrl_k_cast_tma (TMA-staged relayout + RNE cast, push)")
    if info.n_fp8_items:
        kern.append("llrl_k_fp8_tma (fp8 block quant, TMA-staged)")
    roof["kernel"] = " + ".join(kern) + f"; whole sync of GPU {bdev} (binding), CUDA events on its stream"
    roof["t_lb_ms"] = round(t_lb, 3)
    roof["binding_gpu"] = bdev
    if args.replicate == "nccl":
        roof["note"] = "bytes of the fused replica-0 sync only; the NCCL broadcasts come on top"
    if info.nv_amax_read_bytes:
        roof["nv_amax_pass_reread_bytes"] = info.nv_amax_read_bytes
        roof["note"] = ("NVFP4 two-pass sync: achieved counts the algorithmic bytes (each source read once + "
                        "every generator byte written); the per-tensor amax pass re-reads "
                        f"{info.nv_amax_read_bytes / 1e9:.2f} GB on top (in `traffic`, not in `achieved`); "
                        "see nvfp4_supplied_amax for the one-pass sync")
    nv1 = _nv_supplied(job, args, nbytes, peak) if cfg.dst_dtype == "nvfp4" and not args.no_nv_supplied else None

    # end to end through the C ABI with host buffers (pinned), copies in the timed region
    e2e = None
    if not args.no_e2e and args.replicate == "push":   # sync_host has no NCCL-replica stage
        e2e = _e2e(job, args)

    comp = _nccl_comparator(job, args) if (args.comparator and args.gpus > 1) else None
    if args.comparator and args.gpus > 1:
        if cfg.src_dtype == cfg.dst_dtype:                 # copy engines cannot cast
            try:
                comp.update(_ce_comparator(job, args))
            except ImportError as e:                       # cuda-python missing: no CE arm
                comp["ce_memcpy2d_ms"] = None
                comp["ce_error"] = str(e)
        if cfg.fsdp > 1:
            comp.update(_allgather_comparator(job, args))
    ovl = _overlap(job, args) if args.overlap else None

    tot = job.plan.stats()
    tr = job.plan.traffic()
    wire = sum(tr[i][j] for i in range(len(tr)) for j in range(len(tr)) if i != j)
    nvl_per_gpu = max(max(job.plan.device_bytes(d)["nvl_tx"], job.plan.device_bytes(d)["nvl_rx"])
                      for d in range(ndev)) / (ms * 1e6)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "ms_min": round(ms_min, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": f"{cfg.src_dtype}->{cfg.dst_dtype}", "data": DATA,
            "config": config_dict(cfg, args, job.model),
            "throughput": {"gen_bytes_per_s_GB": round(tot.dst_bytes / (ms * 1e6), 1),
                           "algorithmic_bytes_GB": round((tot.src_bytes + tot.dst_bytes) / 1e9, 3),
                           "nvlink_wire_GB": round(wire / 1e9, 3),
                           "nvlink_GBps_per_gpu_max": round(nvl_per_gpu, 1)},
            "roofline": roof,
            "gpu_launches": launches,
            **({"event_floor_us": floor_us} if floor_us is not None else {}),
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if comp:
            line["comparator"] = comp
        if ovl:
            line["overlap"] = ovl
        if nv1:
            line["nvfp4_supplied_amax"] = nv1
        if not args.no_cpu_baseline and args.gpus == 1:      # rank 0 at N=1 only
            job.close()                                     # free the GPU job first (host RAM: pinned e2e)
            line["cpu_baseline"] = cpu_baseline(cfg, args.gpus, single_thread=not args.no_cpu_single)
        print(json.dumps(line), flush=True)
    job.close()
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def _e2e(job, args):
    import torch
    need = sum(t.numel() for t in job.src.values()) + sum(t.numel() for t in job.dst.values())
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    ok = need * local_world < 0.6 * avail
    if _allmax(0.0 if ok else 1.0) > 0:
        return {"value": None, "unit": "ms", "skipped": f"pinned host buffers ({need * local_world / 1e9:.0f} GB "
                f"for this node) exceed 60% of available host RAM ({avail / 1e9:.0f} GB)"}
    host_src = {r: torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for r, t in job.src.items()}
    host_dst = {g: torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for g, t in job.dst.items()}
    for r, t in job.src.items():
        host_src[r].copy_(t)
    steps = max(1, min(args.steps, args.e2e_steps))
    job.sync_host(host_src, host_dst)
    _barrier()
    tot = 0.0
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(job.stream)
        job.sync_host(host_src, host_dst)
        e1.record(job.stream)
        _barrier()                     # step boundary: generator buffers quiescent again
        tot += e0.elapsed_time(e1)
    ms = _allmax(tot / steps)
    h2d = int(_allsum(sum(t.numel() for t in host_src.values())))
    d2h = int(_allsum(sum(t.numel() for t in host_dst.values())))
    return {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps, "api": "llrl_sync_host (C ABI, pinned host buffers)"}


def _caller_nv_amax(job):
    """The caller's side of llrl_sync_nv_amax (e.g. its optimizer epilogue): max |x|
    of every NVFP4 tensor over the trainer regions the plan lists, with torch,
    MAX-reduced over processes.  Not part of the timed sync."""
    import torch
    import torch.distributed as dist
    n = job.plan.nv_num_tensors()
    amax = torch.zeros(max(1, n), dtype=torch.float32, device=torch.device("cuda", job.device))
    dt = torch.float32 if job.cfg.src_dtype == "f32" else torch.bfloat16
    for tid in range(n):
        for s in job.plan.nv_tensor_sources(tid):
            t = job.src.get(s.src_rank)
            if t is not None:
                v = t.view(dt).as_strided((s.rows, s.cols), (s.src_ld, 1), s.src_off)
                amax[tid] = torch.maximum(amax[tid], v.abs().max().float())
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(amax, op=dist.ReduceOp.MAX)
    return amax


def _nv_supplied(job, args, nbytes, peak):
    """NVFP4 through llrl_sync_nv_amax (one pass: the per-tensor amax supplied by
    the caller), timed like the main line (back-to-back, CUDA events, max over
    ranks), against the same algorithmic bytes and peak."""
    import torch
    amax = _caller_nv_amax(job)
    for _ in range(3):
        job.sync_nv_amax(amax)
    _barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, args.steps)
    e0.record(job.stream)
    for _ in range(steps):
        job.sync_nv_amax(amax)
    e1.record(job.stream)
    _barrier()
    ms = _allmax(e0.elapsed_time(e1) / steps)
    ach = nbytes / ms / 1e6
    return {"value": round(ms, 4), "unit": "ms", "steps": steps, "achieved": round(ach, 1), "peak": peak,
            "frac": round(ach / peak, 4), "api": "llrl_sync_nv_amax (C ABI)",
            "amax": "supplied by the caller (here torch max|x| over llrl_plan_nv_tensor_sources, outside the "
                    "timed region -- in an RL step the optimizer epilogue produces it)"}


def _overlap(job, args):
    """NEXT f3: the sync of layer l streams out while the optimizer updates layer
    l+1 (llrl_sync_group per layer group) vs optimizer-then-sync.  The optimizer
    here is a synthetic pass over the trainer bytes of each layer (x * 1.0, one
    read + one write: values unchanged)."""
    import torch
    opt_stream = torch.cuda.Stream(device=job.device)
    n = job.plan.num_groups()
    views = [job.src_group_views(g) for g in range(n)]

    def opt(vs):
        for v in vs:
            v.mul_(1.0)

    def timed(fn, steps=5):
        fn()
        _barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(job.stream)
        for _ in range(steps):
            fn()
        e1.record(job.stream)
        _barrier()
        return _allmax(e0.elapsed_time(e1) / steps)

    def opt_all():
        with torch.cuda.stream(job.stream):
            for g in range(n):
                opt(views[g])

    def sequential():
        opt_all()
        job.sync()

    def overlapped():
        job.overlapped_step(lambda vs: opt(vs), opt_stream)

    out = {"optimizer_only_ms": round(timed(opt_all), 3), "sync_only_ms": round(timed(job.sync), 3),
           "sequential_ms": round(timed(sequential), 3), "overlapped_ms": round(timed(overlapped), 3),
           "groups": n, "optimizer": "synthetic pass x*1.0 over each layer's trainer bytes (torch mul_)"}
    # the same per-layer pipeline captured once in a CUDA graph (device-side completion state)
    graph = torch.cuda.CUDAGraph()
    _barrier()
    with torch.cuda.graph(graph):
        job.overlapped_step(lambda vs: opt(vs), opt_stream, stream=torch.cuda.current_stream())
    out["overlapped_graph_ms"] = round(timed(graph.replay), 3)
    return out


def _nccl_comparator(job, args):
    """NCCL baseline for the same exchange: one all_to_all_single per step moving
    exactly the plan's GPU x GPU byte matrix (already-cast, already-packed bytes;
    a real NCCL solution would add a pack pass before and an unpack pass after)."""
    import torch
    import torch.distributed as dist
    tr = job.plan.traffic()
    me = job.device
    dev = torch.device("cuda", me)
    # chunks of <= 4 GB per GPU (memory-bounded; NCCL runs at full rate on such messages)
    KT = max(1, -(-max(int(sum(tr[me][d] for d in range(args.gpus) if d != me)),
                       int(sum(tr[s_][me] for s_ in range(args.gpus) if s_ != me))) // (4 << 30)))
    KT = int(_allmax(float(KT)))
    send = [0 if d == me else int(tr[me][d]) // KT for d in range(args.gpus)]
    recv = [0 if s_ == me else int(tr[s_][me]) // KT for s_ in range(args.gpus)]
    inp = torch.empty(max(1, sum(send)), dtype=torch.uint8, device=dev)
    out = torch.empty(max(1, sum(recv)), dtype=torch.uint8, device=dev)

    def transport():
        for _ in range(KT):
            dist.all_to_all_single(out[:sum(recv)], inp[:sum(send)], recv, send)

    for _ in range(2):
        transport()
    _barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 10))
    e0.record()
    for _ in range(steps):
        transport()
    e1.record()
    _barrier()
    ms = _allmax(e0.elapsed_time(e1) / steps)
    res = {"nccl_alltoallv_ms": round(ms, 3), "steps": steps,
           "what": f"torch.distributed.all_to_all_single (NCCL) of the plan's off-diagonal byte matrix in {KT} "
                   "chunk(s); transport only, no cast / relayout / pack / unpack"}
    cfg = job.cfg
    if cfg.dst_dtype in ("bf16", "f32") and cfg.src_dtype in ("f32", "bf16"):
        # the whole NCCL pipeline: cast + pack everything sourced here into a send
        # buffer (one torch cast/copy kernel over the trainer bytes), the a2a of the
        # remote part, then unpack everything landing here into the generator buffers
        # (one copy kernel) -- the byte volumes of a pack/unpack solution, without its
        # index arithmetic (a lower bound on that baseline)
        sdt = torch.float32 if cfg.src_dtype == "f32" else torch.bfloat16
        ddt = torch.float32 if cfg.dst_dtype == "f32" else torch.bfloat16
        esd = 4 if cfg.dst_dtype == "f32" else 2
        del inp, out
        torch.cuda.empty_cache()
        # K chunks of at most ~4 GB sent per GPU (memory-bounded, and how a real
        # NCCL pipeline would stream it)
        K = max(1, -(-max(int(sum(tr[me])), int(sum(tr[s_][me] for s_ in range(args.gpus)))) // (4 << 30)))
        K = int(_allmax(float(K)))
        send2 = [0 if d == me else int(tr[me][d]) // K // 16 * 16 for d in range(args.gpus)]
        recv2 = [0 if s_ == me else int(tr[s_][me]) // K // 16 * 16 for s_ in range(args.gpus)]
        r0 = int(tr[me][me]) // K // 16 * 16                 # local part of a chunk (stays on the GPU)
        n_pack = (r0 + sum(send2)) // esd                      # elements packed per chunk
        n_land = r0 + sum(recv2)                               # bytes unpacked per chunk
        # byte volumes are what is timed: read the local trainer buffers and write the
        # local generator buffers cyclically (no extra full-size copies)
        srcs = [t.view(sdt) for t in job.src.values()]
        dsts = list(job.dst.values())

        def span(bufs, k, n):
            """the k-th n-element window over the buffers, cyclically"""
            tot = sum(b.numel() for b in bufs)
            o = (k * n) % max(1, tot)
            for b in bufs:
                if o < b.numel():
                    m = min(n, b.numel() - o)
                    return b[o:o + m]
                o -= b.numel()
            return bufs[0][:0]
        packed = torch.empty(max(1, n_pack), dtype=ddt, device=dev)
        land = torch.empty(max(1, n_land), dtype=torch.uint8, device=dev)

        def pipeline():
            for k in range(K):
                if n_pack:                                      # cast + pack
                    x = span(srcs, k, n_pack)
                    packed[:x.numel()].copy_(x)
                pb = packed.view(torch.uint8)
                dist.all_to_all_single(land[r0:n_land], pb[r0:r0 + sum(send2)], recv2, send2)
                if r0:
                    land[:r0].copy_(pb[:r0])
                if n_land:                                      # unpack
                    y = span(dsts, k, n_land)
                    y.copy_(land[:y.numel()])

        for _ in range(2):
            pipeline()
        _barrier()
        e0.record()
        for _ in range(steps):
            pipeline()
        e1.record()
        _barrier()
        res["nccl_pipeline_ms"] = round(_allmax(e0.elapsed_time(e1) / steps), 3)
        res["pipeline_what"] = (f"{K} chunk(s) of: torch cast+pack of trainer bytes -> NCCL all_to_all_single of "
                                "the remote part -> unpack copy into generator memory (byte volumes only, no index "
                                "math: a lower bound on a pack/NCCL/unpack solution)")
        del packed, land
        return res
    del inp, out
    return res


def _rectangles(runs):
    """Coalesce the plan's canonical 1-D runs (llrl_plan_get_runs, emission order)
    into 2-D copies: maximal sequences of runs of one (param, src rank, dst rank,
    len) whose src and dst offsets advance by constant strides.  Returns arrays
    (src_rank, dst_rank, src_off, dst_off, len, rows, src_step, dst_step) in
    elements; a 1-row rectangle has steps = len."""
    import numpy as np
    n = len(runs)
    if n == 0:
        return [np.zeros(0, np.int64)] * 8
    # one key's runs side by side (the plan interleaves src ranks row by row),
    # emission order kept within a key
    runs = runs[np.lexsort((np.arange(n), runs["len"], runs["dst_rank"], runs["src_rank"], runs["src_param"]))]
    so, do, ln = runs["src_off"], runs["dst_off"], runs["len"]
    key = np.ones(n, bool)                 # key[i]: run i differs in key from run i-1
    key[1:] = ((runs["src_param"][1:] != runs["src_param"][:-1]) | (runs["src_rank"][1:] != runs["src_rank"][:-1])
               | (runs["dst_rank"][1:] != runs["dst_rank"][:-1]) | (ln[1:] != ln[:-1]))
    ds = np.zeros(n, np.int64)
    dd = np.zeros(n, np.int64)
    ds[1:] = so[1:] - so[:-1]
    dd[1:] = do[1:] - do[:-1]
    chg = np.zeros(n, bool)                # delta into run i differs from the delta into run i-1
    chg[2:] = (ds[2:] != ds[1:-1]) | (dd[2:] != dd[1:-1])
    starts = []
    prev_start = -2
    # run i opens a rectangle if its key changes, or its delta breaks the current
    # rectangle's stride (the stride is set by a rectangle's second run: i - 1
    # being a start means run i is that second run, whatever its delta)
    for i in np.nonzero(key | chg)[0].tolist():
        if key[i] or (i - 1 != prev_start):
            starts.append(i)
            prev_start = i
    st = np.array(starts, np.int64)
    en = np.append(st[1:], n)
    rows = en - st
    s_step = np.where(rows > 1, ds[np.minimum(st + 1, n - 1)], ln[st])
    d_step = np.where(rows > 1, dd[np.minimum(st + 1, n - 1)], ln[st])
    return (runs["src_rank"][st].astype(np.int64), runs["dst_rank"][st].astype(np.int64), so[st], do[st], ln[st],
            rows, s_step, d_step)


def _ce_comparator(job, args):
    """Copy-engine baseline on the real tiles (bf16 -> bf16, no cast): every
    rectangle this GPU sources as one cudaMemcpy2DAsync from its trainer buffer
    into the (local or IPC-mapped peer) generator buffer -- what a DMA-engine
    transfer of the same re-layout costs, without any SM work.  The copies are
    captured once in a CUDA graph (thousands of host calls would otherwise bind)
    and the graph replayed per step."""
    import numpy as np
    import torch
    from cuda.bindings import runtime as cr
    cfg = job.cfg
    es = {"bf16": 2, "f32": 4}[cfg.src_dtype]
    sr, dr, so, do, ln, rows, ss, dstep = _rectangles(job.plan.runs())
    mine = np.array([job.src_dev[int(r)] == job.device for r in sr], bool) if len(sr) else np.zeros(0, bool)
    idx = np.nonzero(mine)[0]
    bad = set(idx[(ss[idx] < ln[idx]) | (dstep[idx] < ln[idx])].tolist())   # not a forward 2-D pattern: row by row
    s = torch.cuda.Stream(device=job.device)
    g = torch.cuda.CUDAGraph()
    ncopies = 0
    with torch.cuda.stream(s):
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            h = s.cuda_stream
            for k in idx.tolist():
                sp, dp = job.src_ptrs[int(sr[k])], job.dst_ptrs[int(dr[k])]
                w = int(ln[k]) * es
                if k in bad:
                    for j in range(int(rows[k])):
                        cr.cudaMemcpyAsync(dp + (int(do[k]) + j * int(dstep[k])) * es,
                                           sp + (int(so[k]) + j * int(ss[k])) * es, w,
                                           cr.cudaMemcpyKind.cudaMemcpyDeviceToDevice, h)
                        ncopies += 1
                    continue
                err = cr.cudaMemcpy2DAsync(dp + int(do[k]) * es, int(dstep[k]) * es, sp + int(so[k]) * es,
                                           int(ss[k]) * es, w, int(rows[k]),
                                           cr.cudaMemcpyKind.cudaMemcpyDeviceToDevice, h)[0]
                if err != cr.cudaError_t.cudaSuccess:
                    raise RuntimeError(f"cudaMemcpy2DAsync: {err}")
                ncopies += 1
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    _barrier()
    steps = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(steps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    _barrier()
    ms = _allmax(e0.elapsed_time(e1) / steps)
    del g
    return {"ce_memcpy2d_ms": round(ms, 3), "ce_copies_per_gpu_max": int(_allmax(float(ncopies))),
            "ce_what": "cudaMemcpy2DAsync per rectangle of the plan's runs sourced on each GPU (copy engines, "
                       "peer writes through the IPC mappings), captured in a CUDA graph; no cast, no SM work"}


def _allgather_comparator(job, args):
    """The naive alternative the plan replaces (SURVEY §8(d) "work avoided"):
    every GPU all-gathers each layer group's full trainer bytes (NCCL
    all_gather_into_tensor, per group: memory-bounded), then slices its own
    generator shards out of the gathered copy.  The slice is timed as a plain
    copy of this GPU's generator bytes of the group (byte volume only, no index
    arithmetic), so the result is a lower bound on that baseline."""
    import torch
    import torch.distributed as dist
    p = job.plan
    ng = p.num_groups()
    dev = torch.device("cuda", job.device)
    src_local = [r for r in range(job.S.n_ranks) if job.src_dev[r] == job.device]
    dst_local = [g for g in job.dst if job.dst_dev[g] == job.device]
    chunk = []
    for grp in range(ng):
        mine = sum(max(0, hi - lo) for lo, hi in (p.group_range(0, r, grp) for r in src_local))
        chunk.append(int(_allmax(float(mine))))
    big = max(chunk) if chunk else 0
    send = torch.empty(max(1, big), dtype=torch.uint8, device=dev)
    gath = torch.empty(max(1, big * args.gpus), dtype=torch.uint8, device=dev)
    dst_ranges = [[(g, *p.group_range(1, g, grp)) for g in dst_local] for grp in range(ng)]

    def naive():
        for grp in range(ng):
            c = chunk[grp]
            if c:
                dist.all_gather_into_tensor(gath[:c * args.gpus], send[:c])
            for g, lo, hi in dst_ranges[grp]:
                if hi > lo:
                    job.dst[g][lo:hi].copy_(gath[:hi - lo])

    for _ in range(2):
        naive()
    torch.cuda.synchronize()
    _barrier()
    steps = max(3, min(args.steps, 5))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        naive()
    e1.record()
    torch.cuda.synchronize()
    _barrier()
    ms = _allmax(e0.elapsed_time(e1) / steps)
    del send, gath
    torch.cuda.empty_cache()
    return {"naive_allgather_slice_ms": round(ms, 3), "naive_groups": ng,
            "naive_what": "per layer group: NCCL all_gather_into_tensor of every GPU's trainer bytes of the group "
                          "(padded to the largest), then a copy of this GPU's generator bytes of the group out of "
                          "the gathered buffer (byte volume only: a lower bound on all-gather + slice)"}


def _ncu_traffic(config, n):
    """dram read+write bytes per launch from the committed ncu --set full summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(f"{config}@{n}")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(__import__("synth").CONFIGS))
    ap.add_argument("--impl", default="llrl", choices=["llrl", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-single", action="store_true", help="cpu_baseline: skip the single-threaded pass")
    ap.add_argument("--no-nv-supplied", action="store_true", help="NVFP4: skip the supplied-amax one-pass timing")
    ap.add_argument("--layers", type=int, default=None, help="override decoder layers (profiling only)")
    ap.add_argument("--placement", default=None, choices=["disjoint", "colocated", "rotated", "fanout"])
    ap.add_argument("--multicast", action="store_true", help="NVLS multicast to generator DP replicas (f1)")
    ap.add_argument("--step-sync", action="store_true",
                    help="synchronize + barrier before every timed sync (isolated single-sync latency)")
    ap.add_argument("--replicate", default="push", choices=["push", "nccl"],
                    help="generator DP replicas: fused pushes, or replica 0 + NCCL broadcast (a5)")
    ap.add_argument("--comparator", action="store_true", help="also time an NCCL all-to-all-v of the same bytes")
    ap.add_argument("--overlap", action="store_true", help="also time per-layer optimizer/sync overlap (f3)")
    ap.add_argument("--max-ctas", type=int, default=0, help="cap the sync kernels' CTAs per GPU (0 = all SMs)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_llrl(args)


if __name__ == "__main__":
    main()
