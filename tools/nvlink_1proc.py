"""One process driving several GPUs through the C ABI (single-process comm
setup: llrl_comm_flag_ptr + llrl_comm_set_peer), so that ncu -- which must not
wrap a multi-rank command -- can profile a push kernel that writes a peer's
HBM over NVLink and report its NVLink counters.

  python tools/nvlink_1proc.py [config] [n_gpus] [steps]

Prints the device time per sync (CUDA events, every device's stream, max).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2505_24034_b200 import build  # noqa: E402

build.build()
from paper_2505_24034_b200 import llrl, runner  # noqa: E402
from synth import placement  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    spec = runner.spec_for(name, G)
    cfg, m = spec.cfg, spec.model()
    S, D = llrl.describe(m, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                         cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    sd, dd = placement(cfg, G)
    plan = llrl.Plan(S, D, sd, dd)
    src = {r: torch.empty(S.rank_bytes(r), dtype=torch.uint8, device=f"cuda:{sd[r]}") for r in range(S.n_ranks)}
    dst = {g: torch.empty(D.rank_bytes(g), dtype=torch.uint8, device=f"cuda:{dd[g]}") for g in range(D.n_ranks)}
    streams = [torch.cuda.Stream(device=d) for d in range(G)]
    for r, t in src.items():
        with torch.cuda.device(sd[r]):              # the fill runs on the current device
            llrl.fill_synthetic(S, r, t.data_ptr(), 0, streams[sd[r]].cuda_stream)
    comms = [llrl.Comm(d) for d in range(G)]
    flags = [c.flag_ptr() for c in comms]
    for d in range(G):
        for e in range(G):
            if d != e:
                comms[d].set_peer(e, flags[e])
    sp = [src[r].data_ptr() for r in range(S.n_ranks)]
    dp = [dst[g].data_ptr() for g in range(D.n_ranks)]
    for d in range(G):
        torch.cuda.synchronize(d)

    # NVFP4: the one-pass sync with a supplied per-tensor amax (llrl_sync_nv_amax).
    # The two-pass sync's cross-GPU amax handshake waits on other GPUs' kernels,
    # which ncu's serialisation of the profiled launches would deadlock; the
    # bytes moved are the same (the amax value only changes the codes)
    nv = cfg.dst_dtype == "nvfp4"
    amax = [torch.ones(max(1, plan.nv_num_tensors()), dtype=torch.float32, device=f"cuda:{d}") for d in range(G)] \
        if nv else None

    def one():
        for d in range(G):
            if nv:
                plan.sync_nv_amax(comms[d], d, amax[d].data_ptr(), sp, dp, streams[d].cuda_stream)
            else:
                plan.sync(comms[d], d, sp, dp, streams[d].cuda_stream)

    one()
    for d in range(G):
        torch.cuda.synchronize(d)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(G)]
    for d in range(G):
        ev[d][0].record(streams[d])
    for _ in range(steps):
        one()
    for d in range(G):
        ev[d][1].record(streams[d])
    for d in range(G):
        torch.cuda.synchronize(d)
    ms = max(a.elapsed_time(b) for a, b in ev) / steps
    tr = plan.traffic()
    wire = max(max(sum(tr[i][j] for j in range(G) if j != i), sum(tr[j][i] for j in range(G) if j != i))
               for i in range(G))
    print(f"{name} G={G}: {ms:.3f} ms per sync, max NVLink egress/ingress {wire / 1e9:.2f} GB "
          f"-> {wire / ms / 1e6:.1f} GB/s per GPU")
    for c in comms:
        assert not c.timed_out()
        c.close()
    plan.close()


if __name__ == "__main__":
    main()
