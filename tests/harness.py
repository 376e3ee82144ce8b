"""Test helpers: host trainer buffers from ``synth`` placed by the ORACLE's
layout, and point checks of generator elements / fp8 blocks computed one by
one by the oracle (for full-size configs where the whole oracle is too slow).
Test infrastructure only."""
from __future__ import annotations

import numpy as np

import oracle
import synth


def host_src(ol: oracle.Layout, seed: int):
    """Trainer rank buffers (uint8) filled with synth weights at the oracle's offsets."""
    es = 4 if ol.src_dtype == "f32" else 2
    bufs = []
    for r in range(ol.n_src):
        b = np.zeros(ol.src_rank_bytes(r), np.uint8)
        for p in range(ol.n_src_params):
            off, r0, r1, c0, c1 = ol.src_piece(r, p)
            if r1 <= r0 or c1 <= c0:
                continue
            is_norm = ol.src_param_info(p)[2] == 2
            bits = synth.weight_bits(seed, p, is_norm, ol.src_dtype, np.arange(r0, r1)[:, None], np.arange(c0, c1)[None, :])
            b[off:off + bits.nbytes] = bits.view(np.uint8).reshape(-1)
        bufs.append(b)
    return bufs


def oracle_dst(ol: oracle.Layout, src, sentinel=0):
    dst = [np.full(ol.dst_rank_bytes(g), sentinel, np.uint8) for g in range(ol.n_dst)]
    rc = ol.sync(src, dst)
    assert rc == 0, rc
    return dst


def _src_value_bits(ol, seed, p, row, col):
    is_norm = ol.src_param_info(p)[2] == 2
    return synth.weight_bits(seed, p, is_norm, ol.src_dtype, np.array([row]), np.array([col]))[0]


def expected_elements(ol: oracle.Layout, seed, g, gp, lrs, lcs):
    """bf16 / f32 generator elements (uint16 / uint32 bits) at local coords, one by one."""
    out = []
    for lr, lc in zip(lrs, lcs):
        p, row, col = ol.dst_element_source(g, gp, int(lr), int(lc))
        bits = int(_src_value_bits(ol, seed, p, row, col))
        if ol.src_dtype == "bf16":
            bits <<= 16
        if ol.dst_dtype == "f32":
            out.append(bits)
        else:
            out.append(int(oracle.bf16_rne(np.array([bits], np.uint32))[0]))
    return np.array(out)


def expected_fp8_block(ol: oracle.Layout, seed, g, gp, bi, bj):
    """(codes [rows, cols], scale) of one generator fp8 block, from the oracle."""
    R, C, q, off, soff = ol.dst_param(g, gp)
    r0, c0 = bi * 128, bj * 128
    rows, cols = min(128, R - r0), min(128, C - c0)
    x = np.zeros((rows, cols), np.float32)
    for i in range(rows):
        # one source param per row of a block on every layout we use; resolve per element anyway
        for j in range(cols):
            p, row, col = ol.dst_element_source(g, gp, r0 + i, c0 + j)
            bits = int(_src_value_bits(ol, seed, p, row, col))
            if ol.src_dtype == "bf16":
                bits <<= 16
            x[i, j] = np.array([bits], np.uint32).view(np.float32)[0]
    return oracle.fp8_block(x)


def expected_fp8_block_fast(ol: oracle.Layout, seed, g, gp, bi, bj):
    """Same as expected_fp8_block, resolving the source once per block row segment
    (rows of a 128-wide block map to consecutive columns of one source row)."""
    R, C, q, off, soff = ol.dst_param(g, gp)
    r0, c0 = bi * 128, bj * 128
    rows, cols = min(128, R - r0), min(128, C - c0)
    x = np.zeros((rows, cols), np.float32)
    for i in range(rows):
        p, row, col = ol.dst_element_source(g, gp, r0 + i, c0)
        p2, row2, col2 = ol.dst_element_source(g, gp, r0 + i, c0 + cols - 1)
        assert (p2, row2, col2) == (p, row, col + cols - 1)
        is_norm = ol.src_param_info(p)[2] == 2
        bits = synth.weight_bits(seed, p, is_norm, ol.src_dtype, np.array([row]), np.arange(col, col + cols))
        bits = bits.astype(np.uint32)
        if ol.src_dtype == "bf16":
            bits = bits << np.uint32(16)
        x[i] = bits.view(np.float32)
    return oracle.fp8_block(x)


def expected_mx_group(ol: oracle.Layout, seed, g, gp, r, j):
    """(codes, E8M0 byte) of MXFP8 group j of row r of generator param gp, from the oracle."""
    R, C, q, off, soff = ol.dst_param(g, gp)
    c0 = j * 32
    n = min(32, C - c0)
    p, row, col = ol.dst_element_source(g, gp, r, c0)
    assert ol.dst_element_source(g, gp, r, c0 + n - 1) == (p, row, col + n - 1)
    is_norm = ol.src_param_info(p)[2] == 2
    bits = synth.weight_bits(seed, p, is_norm, ol.src_dtype, np.array([row]), np.arange(col, col + n)).astype(np.uint32)
    if ol.src_dtype == "bf16":
        bits = bits << np.uint32(16)
    return oracle.mx_block(bits.view(np.float32))


def expected_mx4_group(ol: oracle.Layout, seed, g, gp, r, j):
    """(codes one per element, E8M0 byte) of MXFP4 group j of row r, from the oracle."""
    R, C, q, off, soff = ol.dst_param(g, gp)
    c0 = j * 32
    n = min(32, C - c0)
    p, row, col = ol.dst_element_source(g, gp, r, c0)
    is_norm = ol.src_param_info(p)[2] == 2
    bits = synth.weight_bits(seed, p, is_norm, ol.src_dtype, np.array([row]), np.arange(col, col + n)).astype(np.uint32)
    if ol.src_dtype == "bf16":
        bits = bits << np.uint32(16)
    return oracle.mx4_block(bits.view(np.float32))


def dst_tensor_values(ol: oracle.Layout, seed, g, gp):
    """The whole generator-local tensor gp of rank g as fp32 (from synth, row by row
    through the oracle's index mapping) -- for NVFP4's per-tensor scale."""
    R, C, q, off, soff = ol.dst_param(g, gp)
    x = np.zeros((R, C), np.float32)
    for r in range(R):
        p, row, col = ol.dst_element_source(g, gp, r, 0)
        is_norm = ol.src_param_info(p)[2] == 2
        bits = synth.weight_bits(seed, p, is_norm, ol.src_dtype, np.array([row]), np.arange(col, col + C))
        bits = bits.astype(np.uint32)
        if ol.src_dtype == "bf16":
            bits = bits << np.uint32(16)
        x[r] = bits.view(np.float32)
    return x


# ---------------------------------------------------------------- streamed every-byte parity at full size
#
# SURVEY §8(c) "GPU vs oracle: bit-exact byte compare of every dst buffer,
# streamed per layer for 70B/405B".  The trainer buffers are filled on the host
# by the input generator (synth.fast, the C twin of synth.weight_bits) at the
# ORACLE's offsets and copied to the GPU, so neither the product's layout nor
# its fill kernel touches the inputs.  After the sync, every generator
# parameter is recomputed by the oracle (orc_sync_range on one parameter, with
# its trainer pieces regenerated on the host) on a thread pool and compared
# with the GPU's bytes of that parameter's slice of the rank buffer; the slices
# partition each rank buffer, so padding is compared too.  Coverage: a second
# sync over a different sentinel must leave exactly (padding + bytes whose
# expected value equals that sentinel) bytes equal to it.

ALIGN = 256


def _align(x):
    return (x + ALIGN - 1) // ALIGN * ALIGN


def written_extent(ol: oracle.Layout, q, gp):
    """(first byte, end byte, bytes written) of generator param gp on rank q."""
    R, C, quant, off, soff = ol.dst_param(q, gp)
    ddt = ol.dst_dtype
    if not quant:
        n = R * C * {"f32": 4}.get(ddt, 2)
        return off, off + n, n
    data = R * C // 2 if ddt in ("mxfp4", "nvfp4") else R * C
    if ddt == "fp8":
        grid = -(-R // 128) * -(-C // 128) * 4
    elif ddt == "nvfp4":
        grid = R * -(-C // 16)
    else:
        grid = R * -(-C // 32)
    end, n = soff + grid, data + grid
    if ddt == "nvfp4":
        tso = ol.dst_tensor_scale_off(q, gp)
        end, n = tso + 4, n + 4
    return off, end, n


def dst_partition(ol: oracle.Layout, q):
    """[(lo, hi)] per generator param: consecutive slices covering rank q's whole
    buffer (each param's bytes plus the padding after them); and the total
    number of padding bytes."""
    total = ol.dst_rank_bytes(q)
    parts, lo, nwritten = [], 0, 0
    for gp in range(ol.n_dst_params):
        first, end, n = written_extent(ol, q, gp)
        hi = total if gp == ol.n_dst_params - 1 else _align(end) if n else lo
        assert first >= lo or n == 0
        parts.append((lo, hi))
        lo = hi
        nwritten += n
    return parts, total - nwritten


def gp_source_params(ol: oracle.Layout, gp):
    """(first, last) canonical source param feeding generator param gp: the parts
    of a fused tensor are consecutive source params (reading R0), the first part
    at local row 0 and the last at the last row."""
    for q in range(ol.n_dst):
        R, C = ol.dst_param(q, gp)[:2]
        if R * C:
            return ol.dst_element_source(q, gp, 0, 0)[0], ol.dst_element_source(q, gp, R - 1, C - 1)[0]
    return None


def host_src_slice(ol: oracle.Layout, seed, r, p0, p1):
    """Trainer rank r's bytes of source params p0..p1 (synth.fast at the oracle's
    offsets) -> (lo, uint8 buffer of hi - lo bytes), or None if r holds none."""
    from synth import fast
    es = 4 if ol.src_dtype == "f32" else 2
    pieces = []
    for p in range(p0, p1 + 1):
        off, r0, r1, c0, c1 = ol.src_piece(r, p)
        if r1 > r0 and c1 > c0:
            pieces.append((p, off, r0, r1, c0, c1))
    if not pieces:
        return None
    lo = pieces[0][1]
    hi = pieces[-1][1] + (pieces[-1][3] - pieces[-1][2]) * (pieces[-1][5] - pieces[-1][4]) * es
    buf = np.zeros(hi - lo, np.uint8)
    for p, off, r0, r1, c0, c1 in pieces:
        n = (r1 - r0) * (c1 - c0) * es
        fast.fill(buf[off - lo:off - lo + n], seed, p, ol.src_param_info(p)[2] == 2, ol.src_dtype, r0, r1, c0, c1,
                  parallel=False)
    return lo, buf


def fill_src_device(ol: oracle.Layout, seed, src_tensors):
    """Fill the GPU trainer buffers {rank: cuda uint8 tensor} with synth weights
    at the oracle's offsets (host-generated, pinned staging, H2D)."""
    import torch
    from synth import fast
    es = 4 if ol.src_dtype == "f32" else 2
    jobs = []
    for r, t in src_tensors.items():
        assert t.numel() == ol.src_rank_bytes(r)
        for p in range(ol.n_src_params):
            off, r0, r1, c0, c1 = ol.src_piece(r, p)
            if r1 > r0 and c1 > c0:
                jobs.append((t, p, off, r0, r1, c0, c1, (r1 - r0) * (c1 - c0) * es))
    if not jobs:
        return
    cap = min(max(j[-1] for j in jobs), 1 << 30)
    stage = [torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    k = 0
    for t, p, off, r0, r1, c0, c1, n in jobs:
        rows_per = max(1, cap // ((c1 - c0) * es))
        for a in range(r0, r1, rows_per):
            b = min(r1, a + rows_per)
            m = (b - a) * (c1 - c0) * es
            s = k % 2
            if done[s] is not None:
                done[s].synchronize()
            fast.fill(stage[s].numpy()[:m], seed, p, ol.src_param_info(p)[2] == 2, ol.src_dtype, a, b, c0, c1)
            o = off + (a - r0) * (c1 - c0) * es
            t[o:o + m].copy_(stage[s][:m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            done[s] = ev
            k += 1
    torch.cuda.synchronize()


def streamed_compare(ol: oracle.Layout, seed, dst_tensors, sentinel, count_sentinel=None, workers=None,
                     gps=None):
    """Compare every byte of the GPU generator buffers {rank: cuda uint8 tensor}
    (written by a sync over buffers pre-filled with `sentinel`) with the oracle,
    one generator parameter per task on a thread pool.  Returns {rank: bytes of
    the EXPECTED buffer equal to count_sentinel} for the coverage check.
    Raises AssertionError naming the first differing parameter."""
    import concurrent.futures as cf
    import os
    ranks = sorted(dst_tensors)
    parts = {q: dst_partition(ol, q)[0] for q in ranks}
    for q in ranks:
        assert dst_tensors[q].numel() == ol.dst_rank_bytes(q)
    nsrc, ndst = ol.n_src, ol.n_dst
    gps = range(ol.n_dst_params) if gps is None else gps

    def one(gp):
        srcp = gp_source_params(ol, gp)
        slices = {}
        if srcp is not None:
            for r in range(nsrc):
                s = host_src_slice(ol, seed, r, *srcp)
                if s is not None:
                    slices[r] = s
        scratch = np.zeros(1, np.uint8)
        saddr = [slices[r][1].ctypes.data - slices[r][0] if r in slices else scratch.ctypes.data
                 for r in range(nsrc)]
        exp, daddr = {}, []
        for q in range(ndst):
            lo, hi = dst_partition_cache(q)[gp]
            e = np.full(max(1, hi - lo), sentinel, np.uint8)
            exp[q] = (lo, hi, e)
            daddr.append(e.ctypes.data - lo)
        rc = ol.sync_addrs(saddr, daddr, (gp, gp + 1))
        assert rc == 0, f"oracle rc {rc} on generator param {gp}"
        cnt = {}
        for q in ranks:
            lo, hi, e = exp[q]
            if hi == lo:
                cnt[q] = 0
                continue
            got = dst_tensors[q][lo:hi].cpu().numpy()
            e = e[:hi - lo]
            if not np.array_equal(got, e):
                bad = np.nonzero(got != e)[0]
                raise AssertionError(f"generator rank {q} param {gp}: {bad.size} of {hi - lo} bytes differ, "
                                     f"first at byte {lo + int(bad[0])} (got {got[bad[0]]:#x}, want {e[bad[0]]:#x})")
            cnt[q] = int(np.count_nonzero(e == count_sentinel)) if count_sentinel is not None else 0
        return cnt

    _cache = {}

    def dst_partition_cache(q):
        if q not in _cache:
            _cache[q] = parts[q] if q in parts else dst_partition(ol, q)[0]
        return _cache[q]

    for q in range(ndst):          # warm the cache before the threads start
        dst_partition_cache(q)
    if workers is None:
        workers = max(1, min(os.cpu_count() or 1, 16))
    totals = {q: 0 for q in ranks}
    with cf.ThreadPoolExecutor(workers) as ex:
        # biggest parameters first (embed / lm_head) so they do not finish last
        order = sorted(gps, key=lambda gp: -(parts[ranks[0]][gp][1] - parts[ranks[0]][gp][0]))
        for cnt in ex.map(one, order):
            for q, n in cnt.items():
                totals[q] += n
    return totals


def count_equal(t, value, chunk=1 << 31):
    """Bytes of a (GPU) uint8 tensor equal to `value`, in chunks (no full-size temporary)."""
    return sum(int((t[i:i + chunk] == value).sum().item()) for i in range(0, t.numel(), chunk))


def full_parity(ol: oracle.Layout, job, seed=0, s_a=0xA5, s_b=0x5A, workers=None):
    """Every-byte parity of one SyncJob (the launch configuration bench.py
    times) against the oracle, plus exact write coverage.  Returns a dict of
    stage timings (seconds)."""
    import time
    import torch
    t0 = time.perf_counter()
    fill_src_device(ol, seed, job.src)
    t1 = time.perf_counter()
    # run B: coverage count over sentinel s_b
    for t in job.dst.values():
        t.fill_(s_b)
    job.sync()
    torch.cuda.synchronize()
    count_b = {q: count_equal(t, s_b) for q, t in job.dst.items()}
    # run A: the compared sync
    for t in job.dst.values():
        t.fill_(s_a)
    job.sync()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    n_eq_b = streamed_compare(ol, seed, job.dst, s_a, count_sentinel=s_b, workers=workers)
    t3 = time.perf_counter()
    for q in job.dst:
        pad = dst_partition(ol, q)[1]
        assert count_b[q] == n_eq_b[q] + pad, (
            f"generator rank {q}: {count_b[q] - n_eq_b[q] - pad} byte(s) not written by the sync")
    return {"fill_s": t1 - t0, "sync_s": t2 - t1, "compare_s": t3 - t2,
            "bytes": sum(t.numel() for t in job.dst.values())}


def caller_nv_amax(job):
    """What a caller of llrl_sync_nv_amax supplies (e.g. from its optimizer
    epilogue): for every NVFP4 tensor of the plan, max |x| over the trainer
    regions llrl_plan_nv_tensor_sources lists -- here with torch on this
    process's trainer buffers, then a MAX all-reduce across processes.  Test /
    bench side (the caller), not the product."""
    import torch
    import torch.distributed as dist
    plan = job.plan
    n = plan.nv_num_tensors()
    dev = torch.device("cuda", job.device)
    amax = torch.zeros(max(1, n), dtype=torch.float32, device=dev)
    dt = torch.float32 if job.cfg.src_dtype == "f32" else torch.bfloat16
    for tid in range(n):
        for s in plan.nv_tensor_sources(tid):
            t = job.src.get(s.src_rank)
            if t is None:
                continue
            v = t.view(dt).as_strided((s.rows, s.cols), (s.src_ld, 1), s.src_off)
            amax[tid] = torch.maximum(amax[tid], v.abs().max().float())
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(amax, op=dist.ReduceOp.MAX)
    return amax
