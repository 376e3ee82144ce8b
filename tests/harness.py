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
