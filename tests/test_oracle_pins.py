"""Pins of the CPU oracle against things other than itself.

* bf16 RNE: exhaustive over all 2^32 fp32 patterns against ml_dtypes, plus a
  torch CPU sample (two independent library routines); NaN compared as a class
  (reading R6).
* e4m3 (E4M3FN, RN, satfinite): exhaustive over every fp32 with |x| < 464
  against ml_dtypes (non-saturating libraries and satfinite agree there,
  reading R7); saturation checked on the closed form (448).
* fp8 block quantisation: numpy fp32 arithmetic + ml_dtypes cast (tests/brute.py)
  on random and special blocks.
* layout + whole sync: independent brute force (torch.chunk / torch.cat /
  ml_dtypes) over the 80-combination toy sweep and odd layouts; closed-form
  provenance; dst coverage exactly once; generator shards concatenate back to
  cast(full) (round trip with an f32 generator); error codes.
* parameter counts: the public Llama-3.1 sizes (tests/golden/param_counts.txt).
"""
from __future__ import annotations

import concurrent.futures as cf
import os

import ml_dtypes
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import MODELS
from tests import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------- casts

def _bf16_chunk(start, n):
    x = (np.arange(n, dtype=np.uint64) + np.uint64(start)).astype(np.uint32)
    got = oracle.bf16_rne(x)
    with np.errstate(invalid="ignore"):
        ref = x.view(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    nan_in = np.isnan(x.view(np.float32))
    got_nan = ((got & 0x7F80) == 0x7F80) & ((got & 0x7F) != 0)
    bad = (got != ref) & ~nan_in
    return int(bad.sum()), bool(got_nan[nan_in].all())


def test_bf16_rne_exhaustive_vs_ml_dtypes(oracle_lib):
    n = 1 << 24
    with cf.ThreadPoolExecutor(8) as ex:
        res = list(ex.map(lambda s: _bf16_chunk(s, n), range(0, 1 << 32, n)))
    assert sum(r[0] for r in res) == 0
    assert all(r[1] for r in res)


def test_bf16_rne_vs_torch_and_special_cases(oracle_lib):
    rng = np.random.default_rng(1)
    x = rng.integers(0, 1 << 32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    x = x[~np.isnan(x.view(np.float32))]
    ref = torch.from_numpy(x.view(np.float32).copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(oracle.bf16_rne(x), ref)
    # SURVEY App. B probes: ties to even, subnormal rounding, overflow to Inf
    cases = {0x3F808000: 0x3F80, 0x3F818000: 0x3F82, 0x00038000: 0x0004, 0x7F7F8000: 0x7F80,
             0x80008000: 0x8000, 0x00008001: 0x0001, 0x7F7FFFFF: 0x7F80, 0xFF800000: 0xFF80}
    for k, v in cases.items():
        assert oracle.bf16_rne(np.array([k], np.uint32))[0] == v, hex(k)


def _e4m3_chunk(start, n):
    x = (np.arange(n, dtype=np.uint64) + np.uint64(start)).astype(np.uint32)
    f = x.view(np.float32)
    keep = np.abs(f) < 464
    f = f[keep]
    got = oracle.e4m3(f)
    ref = f.astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
    return int((got != ref).sum())


def test_e4m3_exhaustive_below_464_vs_ml_dtypes(oracle_lib):
    limit = int(np.array([464.0], np.float32).view(np.uint32)[0])   # 0x43E80000
    n = 1 << 24
    starts = list(range(0, limit, n)) + list(range(0x80000000, 0x80000000 + limit, n))
    with cf.ThreadPoolExecutor(8) as ex:
        assert sum(ex.map(lambda s: _e4m3_chunk(s, n), starts)) == 0


def test_e4m3_saturation_and_specials(oracle_lib):
    f = np.array([448.0, 449.0, 464.0, 465.0, 1e30, -1e30, -500.0, 2.0 ** -10, 1.5 * 2.0 ** -10,
                  2.0 ** -9, -2.0 ** -9, 2.0 ** -6, 0.0, -0.0, 1e-45, -1e-45], np.float32)
    want = [0x7E, 0x7E, 0x7E, 0x7E, 0x7E, 0xFE, 0xFE, 0x00, 0x01, 0x01, 0x81, 0x08, 0x00, 0x80, 0x00, 0x80]
    assert oracle.e4m3(f).tolist() == want
    assert oracle.e4m3(np.array([np.nan], np.float32))[0] & 0x7F == 0x7F


@pytest.mark.parametrize("kind", ["random", "zero", "outlier", "ties", "subnormal_out", "partial", "tiny"])
def test_fp8_block_vs_numpy_ml_dtypes(oracle_lib, kind):
    rng = np.random.default_rng(7)
    shape = (128, 128)
    if kind == "random":
        x = rng.normal(0, 0.02, shape).astype(np.float32)
    elif kind == "zero":
        x = np.zeros(shape, np.float32)
        x[3, 5] = -0.0
    elif kind == "outlier":
        x = rng.normal(0, 0.02, shape).astype(np.float32)
        x[17, 99] = -37.5
    elif kind == "ties":
        # amax 448 -> inv = 1: values exactly halfway between e4m3 neighbours
        x = rng.choice(np.array([1.0625, 1.1875, 2.125, 3.25, 9.5, 0.0029296875, -1.0625, 448.0], np.float32), shape)
    elif kind == "subnormal_out":
        x = rng.normal(0, 1e-4, shape).astype(np.float32)
        x[0, 0] = 1.0
    elif kind == "partial":
        shape = (64, 96)
        x = rng.normal(0, 0.02, shape).astype(np.float32)
    else:  # amax below the 2^-64 floor
        x = (rng.normal(0, 1, shape) * 1e-30).astype(np.float32)
    q, s = oracle.fp8_block(x)
    q_ref, s_ref = brute.fp8_quant(x)
    assert s == s_ref[0, 0]
    assert np.array_equal(q, q_ref)


@pytest.mark.parametrize("kind", ["random", "wide_range", "zero", "saturating", "subnormal", "partial"])
def test_mx_block_vs_numpy_ml_dtypes(oracle_lib, kind):
    """MXFP8 (R13): oracle vs numpy frexp / ml_dtypes; the scale byte decodes,
    as ml_dtypes float8_e8m0fnu, to the power of two the block was divided by."""
    rng = np.random.default_rng(11)
    n = 32
    if kind == "random":
        x = rng.normal(0, 0.02, (64, n)).astype(np.float32)
    elif kind == "wide_range":
        x = (rng.normal(0, 1, (64, n)) * 10.0 ** rng.uniform(-37, 37, (64, 1))).astype(np.float32)
    elif kind == "zero":
        x = np.zeros((4, n), np.float32)
        x[1, 3] = -0.0
    elif kind == "saturating":   # amax mantissa >= 1.75: largest elements scale into (448, 512)
        x = rng.uniform(-1, 1, (64, n)).astype(np.float32)
        x[:, 0] = np.float32(1.96875)
    elif kind == "subnormal":
        x = (rng.normal(0, 1, (64, n)) * 1e-39).astype(np.float32)
    else:
        n = 20
        x = rng.normal(0, 0.02, (8, n)).astype(np.float32)
    qb, sb = brute.mx_quant(x)
    for r in range(x.shape[0]):
        q, sc = oracle.mx_block(x[r])
        assert sc == sb[r, 0]
        assert np.array_equal(q, qb[r])
        amax = np.abs(x[r]).max()
        scale = float(np.array([sc], np.uint8).view(ml_dtypes.float8_e8m0fnu).astype(np.float64)[0])
        if amax > 0 and sc > 0:
            assert 256 <= amax / scale < 512          # floor(log2 amax) - 8 == log2 scale
    if kind == "saturating":
        assert (qb[:, 0] & 0x7F == 0x7E).all()        # 1.96875 * 2^8 = 504 -> satfinite 448


def _e2m1_chunk(start, n):
    x = (np.arange(n, dtype=np.uint64) + np.uint64(start)).astype(np.uint32)
    f = x.view(np.float32)
    f = f[np.isfinite(f)]
    return int((oracle.e2m1(f) != f.astype(ml_dtypes.float4_e2m1fn).view(np.uint8)).sum())


def test_e2m1_exhaustive_below_8_vs_ml_dtypes(oracle_lib):
    """E2M1 (R15): every fp32 with |x| < 8 (both signs) against ml_dtypes
    float4_e2m1fn (RNE, saturating at 6), plus the closed-form grid."""
    limit = int(np.array([8.0], np.float32).view(np.uint32)[0])
    n = 1 << 24
    starts = list(range(0, limit, n)) + list(range(0x80000000, 0x80000000 + limit, n))
    with cf.ThreadPoolExecutor(8) as ex:
        assert sum(ex.map(lambda s: _e2m1_chunk(s, n), starts)) == 0
    f = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 7.0, 1e30, -0.25, 0.5, 6.0], np.float32)
    assert oracle.e2m1(f).tolist() == [0, 2, 2, 4, 4, 6, 6, 7, 7, 8, 1, 7]


@pytest.mark.parametrize("kind", ["random", "wide_range", "zero", "saturating", "partial"])
def test_mx4_block_vs_numpy_ml_dtypes(oracle_lib, kind):
    rng = np.random.default_rng(12)
    n = 32
    if kind == "random":
        x = rng.normal(0, 0.02, (64, n)).astype(np.float32)
    elif kind == "wide_range":
        x = (rng.normal(0, 1, (64, n)) * 10.0 ** rng.uniform(-37, 37, (64, 1))).astype(np.float32)
    elif kind == "zero":
        x = np.zeros((4, n), np.float32)
    elif kind == "saturating":   # amax mantissa >= 1.5: largest elements scale into (6, 8)
        x = rng.uniform(-1, 1, (64, n)).astype(np.float32)
        x[:, 0] = np.float32(1.875)
    else:
        n = 20
        x = rng.normal(0, 0.02, (8, n)).astype(np.float32)
    packed, sb = brute.mx4_quant(x)
    for r in range(x.shape[0]):
        q, sc = oracle.mx4_block(x[r])
        assert sc == sb[r, 0]
        qq = np.zeros(n + (n & 1), np.uint8)
        qq[:n] = q
        assert np.array_equal((qq[0::2] | (qq[1::2] << 4)).astype(np.uint8), packed[r])


@pytest.mark.parametrize("kind", ["random", "zero_groups", "outlier", "tiny", "wide_range", "partial"])
def test_nvfp4_vs_numpy_ml_dtypes(oracle_lib, kind):
    """NVFP4 (R16): per-tensor and per-group scales vs numpy fp32 + ml_dtypes;
    'outlier' drives most group scales into E4M3 subnormals, 'zero_groups' the
    s_q = 0 branch, 'tiny' the 2^-64 amax floor."""
    rng = np.random.default_rng(13)
    R, C = 16, 64
    x = rng.normal(0, 0.02, (R, C)).astype(np.float32)
    if kind == "zero_groups":
        x[:, 16:32] = 0
        x[3] = 0
    elif kind == "outlier":
        x[5, 7] = 1e4
    elif kind == "tiny":
        x = (x * 1e-30).astype(np.float32)
    elif kind == "wide_range":
        x = (x * 10.0 ** rng.uniform(-20, 20, (R, 1))).astype(np.float32)
    elif kind == "partial":
        x = x[:, :40]
        C = 40
    packed, sb, ts = brute.nv_quant(x)
    dec, enc = oracle.nv_tensor_scales(x)
    assert dec == ts[0]
    for r in range(R):
        for j in range(-(-C // 16)):
            q, sc = oracle.nv_group(x[r, j * 16:(j + 1) * 16], enc)
            assert sc == sb[r, j], (r, j)
            qq = np.zeros(len(q) + (len(q) & 1), np.uint8)
            qq[:len(q)] = q
            assert np.array_equal((qq[0::2] | (qq[1::2] << 4)).astype(np.uint8),
                                  packed[r, j * 8:j * 8 + len(qq) // 2]), (r, j)


# --------------------------------------------------------------------------- layout / sync

def _run_oracle(m, fsdp, tpt, tpg, sdt, ddt, inner, src, sentinel=0):
    L = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, inner)
    assert L.status == 0
    dst = [np.full(L.dst_rank_bytes(g), sentinel, np.uint8) for g in range(tpg)]
    rc = L.sync(src, dst)
    assert rc == 0, rc
    return L, dst


SWEEP = [(f, tt, tg) for f in (1, 2, 3, 4, 8) for tt in (1, 2, 4, 8) for tg in (1, 2, 4, 8)]


@pytest.mark.parametrize("fsdp,tpt,tpg", SWEEP)
def test_oracle_vs_brute_toy_sweep_bf16(oracle_lib, fsdp, tpt, tpg):
    m = MODELS["toy"].replace(n_layers=1)
    src, want = brute.build(m, 3, fsdp, tpt, tpg, "f32", "bf16")
    L = oracle.Layout(m, fsdp, tpt, tpg, "f32", "bf16")
    assert [L.src_rank_bytes(r) for r in range(fsdp * tpt)] == [b.size for b in src]
    _, dst = _run_oracle(m, fsdp, tpt, tpg, "f32", "bf16", False, src)
    assert [d.size for d in dst] == [w.size for w in want]
    for d, w in zip(dst, want):
        assert np.array_equal(d, w)


@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt,inner", [
    (2, 1, 2, "f32", "bf16", False),      # C1
    (3, 1, 4, "f32", "fp8", False),       # multi-source fp8 blocks
    (2, 2, 8, "bf16", "fp8", False),      # multi-source blocks + KV replication
    (2, 2, 8, "bf16", "fp8", True),       # FSDP-innermost mesh
    (1, 8, 8, "bf16", "fp8", False),      # C4 shape class
    (8, 1, 8, "bf16", "bf16", False),     # C3 shape class
    (2, 4, 8, "bf16", "bf16", False),     # C5 shape class
    (2, 4, 8, "bf16", "bf16", True),
    (3, 2, 4, "f32", "f32", False),       # identity cast (provenance mode)
    (4, 1, 1, "f32", "bf16", False),
    (3, 1, 4, "f32", "mxfp8", False),     # MXFP8 (R13)
    (2, 2, 8, "bf16", "mxfp8", True),
    (1, 8, 8, "bf16", "mxfp8", False),
    (3, 1, 4, "f32", "mxfp4", False),     # MXFP4 (R15)
    (2, 2, 8, "bf16", "mxfp4", True),
    (2, 1, 2, "f32", "nvfp4", False),     # NVFP4 (R16)
    (2, 2, 8, "bf16", "nvfp4", True),
])
def test_oracle_vs_brute_odd_layouts(oracle_lib, fsdp, tpt, tpg, sdt, ddt, inner):
    m = MODELS["toy"]
    src, want = brute.build(m, 5, fsdp, tpt, tpg, sdt, ddt, inner)
    _, dst = _run_oracle(m, fsdp, tpt, tpg, sdt, ddt, inner, src)
    for d, w in zip(dst, want):
        assert np.array_equal(d, w)


@pytest.mark.parametrize("fsdp,tpt,tpg,dp,sdt,ddt", [(4, 1, 1, 4, "f32", "bf16"), (2, 2, 2, 3, "bf16", "fp8"),
                                                    (3, 1, 4, 2, "f32", "fp8")])
def test_oracle_vs_brute_generator_dp(oracle_lib, fsdp, tpt, tpg, dp, sdt, ddt):
    """Generator DP replicas (R12): every replica is a byte copy of its TP rank."""
    m = MODELS["toy"]
    src, want = brute.build(m, 6, fsdp, tpt, tpg, sdt, ddt, dp_gen=dp)
    L = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, False, dp)
    assert L.status == 0 and L.n_dst == tpg * dp
    dst = [np.zeros(L.dst_rank_bytes(q), np.uint8) for q in range(L.n_dst)]
    assert L.sync(src, dst) == 0
    for d, w in zip(dst, want):
        assert np.array_equal(d, w)


@pytest.mark.parametrize("fsdp,tpt,ppt,tpg,ppg,dp,sdt,ddt", [
    (2, 1, 2, 2, 1, 1, "f32", "bf16"),     # trainer PP=2 -> generator without PP
    (1, 2, 1, 2, 2, 1, "bf16", "fp8"),     # generator PP=2
    (3, 1, 2, 4, 2, 2, "f32", "mxfp8"),    # both sides staged, with DP replicas
])
def test_oracle_vs_brute_pipeline_stages(oracle_lib, fsdp, tpt, ppt, tpg, ppg, dp, sdt, ddt):
    """Decoupled pipeline parallelism (R14): layer -> stage maps differ per side."""
    m = MODELS["toy"]
    src, want = brute.build(m, 21, fsdp, tpt, tpg, sdt, ddt, dp_gen=dp, pp_train=ppt, pp_gen=ppg)
    L = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, False, dp, ppt, ppg)
    assert L.status == 0 and L.n_src == len(src) and L.n_dst == len(want)
    assert [L.src_rank_bytes(r) for r in range(L.n_src)] == [b.size for b in src]
    dst = [np.zeros(L.dst_rank_bytes(q), np.uint8) for q in range(L.n_dst)]
    assert L.sync(src, dst) == 0
    for d, w in zip(dst, want):
        assert np.array_equal(d, w)
    assert oracle.Layout(m, 1, 1, 1, sdt, ddt, False, 1, 3, 1).status == oracle.E_INDIVISIBLE   # 2 layers / 3


def test_oracle_provenance_closed_form(oracle_lib):
    """f32 -> f32 identity: every generator element equals the generator value of
    the source coordinate given in closed form by readings R4 (no brute force)."""
    m = MODELS["toy"]
    fsdp, tpt, T = 3, 2, 8
    src, _ = brute.build(m, 11, fsdp, tpt, T, "f32", "f32")
    L, dst = _run_oracle(m, fsdp, tpt, T, "f32", "f32", False, src)
    hd, H, KV, d, f, V = m.head_dim, m.n_heads, m.n_kv_heads, m.d_model, m.d_ffn, m.vocab
    for g in range(T):
        for gp in range(L.n_dst_params):
            R, C, _, off, _ = L.dst_param(g, gp)
            got = dst[g][off:off + R * C * 4].view(np.uint32).reshape(R, C)
            rr = np.arange(R)[:, None]
            cc = np.arange(C)[None, :]
            # generator param gp -> (source param(s), closed-form coordinates)
            if gp == 0:                       # embed: vocab rows g*V/T + r
                exp = synth.weight_bits(11, 0, False, "f32", g * (V // T) + rr, cc)
            elif gp == L.n_dst_params - 2:    # final_norm
                exp = synth.weight_bits(11, L.n_src_params - 2, True, "f32", rr, cc)
            elif gp == L.n_dst_params - 1:    # lm_head
                exp = synth.weight_bits(11, L.n_src_params - 1, False, "f32", g * (V // T) + rr, cc)
            else:
                l, s = divmod(gp - 1, 6)
                base = 1 + 9 * l
                if s in (0, 3):               # norms: full copy
                    exp = synth.weight_bits(11, base + (0 if s == 0 else 5), True, "f32", rr, cc)
                elif s == 1:                  # qkv
                    qr = H * hd // T
                    head = g // (T // KV)     # T > KV here: replicated whole KV head
                    exp = np.where(rr < qr, synth.weight_bits(11, base + 1, False, "f32", g * qr + rr, cc),
                                   np.where(rr < qr + hd,
                                            synth.weight_bits(11, base + 2, False, "f32", head * hd + rr - qr, cc),
                                            synth.weight_bits(11, base + 3, False, "f32", head * hd + rr - qr - hd, cc)))
                elif s == 2:                  # o: input columns g*H*hd/T + c
                    exp = synth.weight_bits(11, base + 4, False, "f32", rr, g * (H * hd // T) + cc)
                elif s == 4:                  # gate_up
                    fr = f // T
                    exp = np.where(rr < fr, synth.weight_bits(11, base + 6, False, "f32", g * fr + rr, cc),
                                   synth.weight_bits(11, base + 7, False, "f32", g * fr + rr - fr, cc))
                else:                         # down
                    exp = synth.weight_bits(11, base + 8, False, "f32", rr, g * (f // T) + cc)
            assert np.array_equal(got, exp), (g, gp)


def test_oracle_dst_coverage_exactly_once(oracle_lib):
    """Two runs with different sentinels: bytes that differ were never written.
    They must be exactly the alignment padding between parameter pieces."""
    m = MODELS["toy"]
    for cfg in [(3, 2, 8, "bf16", "fp8"), (2, 1, 2, "f32", "bf16")]:
        src, _ = brute.build(m, 2, cfg[0], cfg[1], cfg[2], cfg[3], cfg[4])
        L, a = _run_oracle(m, *cfg, False, src, sentinel=0x00)
        _, b = _run_oracle(m, *cfg, False, src, sentinel=0xFF)
        for g in range(cfg[2]):
            covered = np.zeros(a[g].size, bool)
            for gp in range(L.n_dst_params):
                R, C, q, off, soff = L.dst_param(g, gp)
                es = 1 if q else {"f32": 4, "bf16": 2, "fp8": 2}[cfg[4]]
                assert not covered[off:off + R * C * es].any()
                covered[off:off + R * C * es] = True
                if q:
                    n = -(-R // 128) * -(-C // 128) * 4
                    assert not covered[soff:soff + n].any()
                    covered[soff:soff + n] = True
            written = a[g] == b[g]
            assert np.array_equal(written, covered)


def test_oracle_errors(oracle_lib):
    m = MODELS["toy"]
    assert oracle.Layout(m, 1, 1, 3, "f32", "bf16").status == oracle.E_INDIVISIBLE     # H % 3
    assert oracle.Layout(m, 1, 1, 16, "f32", "bf16").status == oracle.E_INDIVISIBLE    # H=8 % 16
    assert oracle.Layout(m, 1, 3, 2, "f32", "bf16").status == oracle.E_INDIVISIBLE     # trainer TP 3
    assert oracle.Layout(m, 1, 1, 2, "bf16", "f32").status == oracle.E_UNSUPPORTED
    # replicas that differ: norms are replicated over trainer TP ranks
    src, _ = brute.build(m, 1, 1, 2, 2, "f32", "bf16")
    L = oracle.Layout(m, 1, 2, 2, "f32", "bf16")
    off = L.src_piece(1, 1)[0]                # l0.attn_norm on rank 1
    src[1][off] ^= 1
    dst = [np.zeros(L.dst_rank_bytes(g), np.uint8) for g in range(2)]
    assert L.sync(src, dst) == oracle.E_MISMATCH


def test_param_counts_match_public_llama_sizes(oracle_lib):
    """tests/golden/param_counts.txt: Llama-3.1 public parameter counts [ext]
    (SURVEY.md §8 shapes table); the oracle's parameter list must sum to them."""
    for line in open(os.path.join(GOLDEN, "param_counts.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        name, count = line.split()
        L = oracle.Layout(MODELS[name], 1, 1, 1)
        total = sum(L.src_param_info(p)[0] * L.src_param_info(p)[1] for p in range(L.n_src_params))
        assert total == int(count), name


# --------------------------------------------------------------------------- invariants (SURVEY §8(c) pins iii)

@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt", [
    (2, 1, 4, "f32", "bf16"),      # KV replication (tp_gen 4 > KV 2)
    (3, 2, 2, "bf16", "bf16"),
    (4, 1, 1, "f32", "f32"),       # identity: round trip trainer -> generator -> full
    (2, 2, 8, "f32", "f32"),
    (1, 1, 8, "bf16", "bf16"),
])
def test_oracle_generator_shards_concatenate_to_cast_full(oracle_lib, fsdp, tpt, tpg, sdt, ddt):
    """Un-fusing every generator rank's qkv / gate_up and concatenating the shards
    along the split dimension gives cast(full(p)) for every parameter; norms are
    full copies on every rank; with tp_gen > KV each rank's k / v is its head
    group's slice.  With an f32 generator this is the round trip
    trainer shards -> generator shards -> the full tensor the trainer shards were
    cut from.  Independent of brute.py's per-rank slicing: here the full tensors
    are rebuilt from the oracle's output."""
    m = MODELS["toy"]
    seed = 23
    ol = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt)
    dst = harness_oracle_dst(ol, seed)
    full = brute.full_tensors(m, seed, sdt)
    if ddt == "bf16" and sdt == "f32":
        cast = {k: v.view(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16) for k, v in full.items()}
    else:
        cast = full
    odt = np.uint16 if ddt == "bf16" else np.uint32
    es = np.dtype(odt).itemsize

    def tensor(g, gp):
        R, C, q, off, _ = ol.dst_param(g, gp)
        assert q == 0
        return dst[g][off:off + R * C * es].view(odt).reshape(R, C)

    H, KV, hd = m.n_heads, m.n_kv_heads, m.head_dim
    qr = H * hd // tpg
    kvr = hd if tpg > KV else KV * hd // tpg
    gps = ["embed"] + [f"l{l}.{n}" for l in range(m.n_layers)
                       for n in ("attn_norm", "qkv", "o", "mlp_norm", "gate_up", "down")] + ["final_norm", "lm_head"]
    assert len(gps) == ol.n_dst_params
    for gp, name in enumerate(gps):
        shards = [tensor(g, gp) for g in range(tpg)]
        base = name.split(".")[-1]
        pre = name[:-len(base)]
        if base in ("attn_norm", "mlp_norm", "final_norm"):
            for s in shards:
                assert np.array_equal(s.reshape(-1), cast[name].reshape(-1)), name
        elif base in ("embed", "lm_head"):
            assert np.array_equal(np.concatenate(shards, 0), cast[name]), name
        elif base in ("o", "down"):
            assert np.array_equal(np.concatenate(shards, 1), cast[name]), name
        elif base == "gate_up":
            f = m.d_ffn // tpg
            assert np.array_equal(np.concatenate([s[:f] for s in shards], 0), cast[pre + "gate"]), name
            assert np.array_equal(np.concatenate([s[f:] for s in shards], 0), cast[pre + "up"]), name
        else:                                   # qkv
            assert np.array_equal(np.concatenate([s[:qr] for s in shards], 0), cast[pre + "q"]), name
            for j, kv in enumerate(("k", "v")):
                parts = [s[qr + j * kvr:qr + (j + 1) * kvr] for s in shards]
                if tpg > KV:                    # rank g holds head g // (tpg / KV)
                    rep = tpg // KV
                    for g in range(tpg):
                        h = g // rep
                        assert np.array_equal(parts[g], cast[pre + kv][h * hd:(h + 1) * hd]), (name, kv, g)
                    parts = parts[::rep]
                assert np.array_equal(np.concatenate(parts, 0), cast[pre + kv]), (name, kv)


def harness_oracle_dst(ol, seed):
    from tests import harness
    return harness.oracle_dst(ol, harness.host_src(ol, seed))


# --------------------------------------------------------------------------- point-check helpers

def _id_tensors(m):
    """Full tensors whose element bits are a global element id (param-major,
    row-major): decoding a generator element's bits gives its source coordinate."""
    full, starts, shapes = {}, [], []
    base = 0
    for pid, (name, R, C, split) in enumerate(brute.src_params(m)):
        full[name] = (np.arange(R * C, dtype=np.uint64) + np.uint64(base)).astype(np.uint32).reshape(R, C)
        starts.append(base)
        shapes.append((R, C))
        base += R * C
    assert base < 2 ** 32
    return full, np.array(starts, np.int64), shapes


def _decode_ids(ids, starts, shapes):
    pid = np.searchsorted(starts, ids.astype(np.int64), side="right") - 1
    cols = np.array([c for _, c in shapes], np.int64)[pid]
    loc = ids.astype(np.int64) - starts[pid]
    return pid, loc // cols, loc % cols


ELEM_SRC_CASES = ([(f, tt, tg, 1, 1, 1, False) for f in (1, 2, 3, 4, 8) for tt in (1, 2, 4, 8) for tg in (1, 2, 4, 8)]
                  + [(2, 2, 8, 1, 1, 1, True), (3, 1, 4, 3, 1, 1, False), (2, 1, 2, 1, 2, 1, False),
                     (1, 2, 2, 1, 1, 2, False), (3, 1, 4, 2, 2, 2, False)])


@pytest.mark.parametrize("fsdp,tpt,tpg,dp,ppt,ppg,inner", ELEM_SRC_CASES)
def test_dst_element_source_vs_brute(oracle_lib, fsdp, tpt, tpg, dp, ppt, ppg, inner):
    """orc_dst_element_source (the index map every full-size point check relies
    on), for EVERY element of every generator param of every rank, against the
    independent brute force: tensors whose bits are their own global element id,
    re-split by brute.generator_pieces (torch.chunk / np.concatenate, readings
    R4, R12, R14) in identity (f32) mode, then decoded."""
    m = MODELS["toy"]
    full, starts, shapes = _id_tensors(m)
    ranks = brute.generator_pieces(m, full, tpg, "f32", "f32", ppg, grouped=True)
    L = oracle.Layout(m, fsdp, tpt, tpg, "f32", "f32", inner, dp, ppt, ppg)
    assert L.status == 0
    for q in range(L.n_dst):
        tensors = ranks[q % (tpg * ppg)]
        assert len(tensors) == L.n_dst_params
        for gp in range(L.n_dst_params):
            want = tensors[gp][0].view(np.uint32)
            R, C = L.dst_param(q, gp)[:2]
            assert want.size == R * C, (q, gp)
            if R * C == 0:
                continue
            p, r, c = L.dst_param_sources(q, gp)
            wp, wr, wc = _decode_ids(want.reshape(R, C), starts, shapes)
            assert np.array_equal(p, wp) and np.array_equal(r, wr) and np.array_equal(c, wc), (q, gp)
            # the scalar entry point agrees with the vector one on the corners
            for lr, lc in ((0, 0), (R - 1, C - 1), (R // 2, C // 3)):
                assert L.dst_element_source(q, gp, lr, lc) == (p[lr, lc], r[lr, lc], c[lr, lc])


@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt,dp,ppg", [
    (2, 1, 2, "f32", "nvfp4", 1, 1), (2, 2, 8, "bf16", "nvfp4", 1, 1), (3, 1, 4, "bf16", "nvfp4", 2, 1),
    (1, 2, 2, "bf16", "nvfp4", 1, 2), (3, 1, 4, "f32", "fp8", 1, 1), (2, 2, 8, "bf16", "mxfp8", 1, 1),
    (3, 1, 4, "f32", "mxfp4", 1, 2), (2, 1, 2, "f32", "bf16", 1, 1)])
def test_dst_offsets_vs_brute_packing(oracle_lib, fsdp, tpt, tpg, sdt, ddt, dp, ppg):
    """orc_dst_param's data / scale-grid offsets and orc_dst_tensor_scale_off (the
    NVFP4 fp32 tensor scale every full-size check reads) against brute.py's own
    walk of the generator tensors (reading R0, R9, R16): codes, scale grid and
    tensor scale each at the next 256-byte boundary."""
    m = MODELS["toy"]
    full = brute.full_tensors(m, 3, sdt)
    ranks = brute.generator_pieces(m, full, tpg, sdt, ddt, ppg, grouped=True)
    L = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, False, dp, 1, ppg)
    assert L.status == 0
    for q in range(L.n_dst):
        tensors = ranks[q % (tpg * ppg)]
        offs, total = brute.offsets([a for grp in tensors for a in grp])
        assert L.dst_rank_bytes(q) == total
        k = 0
        for gp, grp in enumerate(tensors):
            R, C, quant, off, soff = L.dst_param(q, gp)
            assert off == offs[k], (q, gp)
            assert quant == (len(grp) > 1)
            assert soff == (offs[k + 1] if len(grp) > 1 else -1), (q, gp)
            assert L.dst_tensor_scale_off(q, gp) == (offs[k + 2] if len(grp) == 3 else -1), (q, gp)
            k += len(grp)
