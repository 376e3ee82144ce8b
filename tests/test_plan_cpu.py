"""Host logic of the product (no GPU): the C ABI loads and exports every symbol
include/llrl.h declares; the product's layouts equal the oracle's; the plan's
canonical runs cover every generator element exactly once and, executed by a
test-only CPU interpreter, reproduce the oracle's bytes; the plan's traffic
and byte counts match SURVEY.md App. A / BASELINE.md §3 [derived] figures.
"""
from __future__ import annotations

import os
import re

import ml_dtypes
import numpy as np
import pytest

import oracle
from synth import MODELS, CONFIGS, placement
from tests import brute

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2505_24034_b200 import build
    build.build()
    from paper_2505_24034_b200 import llrl
    return llrl


def test_library_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "llrl.h")).read()
    declared = set(re.findall(r"^(?:llrl_status|void|const char \*)\s*(llrl_[a-z0-9_]+)\(", hdr, re.M))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L.lib(), name), name
    assert set(L.EXPORTS) == declared


@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt,inner", [
    (f, tt, tg, "f32", "bf16", False) for f in (1, 2, 3, 4, 8) for tt in (1, 2, 4, 8) for tg in (1, 2, 4, 8)
] + [(2, 2, 8, "bf16", "fp8", True), (3, 1, 4, "f32", "fp8", False), (3, 2, 4, "f32", "f32", False),
      (3, 1, 4, "f32", "mxfp8", False), (2, 2, 8, "bf16", "mxfp8", True), (3, 1, 4, "f32", "mxfp4", False),
      (2, 2, 8, "bf16", "mxfp4", True), (2, 1, 2, "f32", "nvfp4", False), (2, 2, 8, "bf16", "nvfp4", True)])
def test_layout_matches_oracle(L, fsdp, tpt, tpg, sdt, ddt, inner):
    m = MODELS["toy"]
    S, D = L.describe(m, fsdp, tpt, tpg, sdt, ddt, inner)
    O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, inner)
    assert S.n_params == O.n_src_params and D.n_params == O.n_dst_params
    for r in range(S.n_ranks):
        assert S.rank_bytes(r) == O.src_rank_bytes(r)
        for p in range(S.n_params):
            v = S.param_view(r, p)
            off, r0, r1, c0, c1 = O.src_piece(r, p)
            assert (v.byte_off, v.full_r0, v.full_r0 + v.rows, v.full_c0, v.full_c0 + v.cols) == (off, r0, r1, c0, c1)
    for g in range(D.n_ranks):
        assert D.rank_bytes(g) == O.dst_rank_bytes(g)
        for gp in range(D.n_params):
            v = D.param_view(g, gp)
            assert (v.rows, v.cols, v.quantised, v.byte_off, v.scale_off) == O.dst_param(g, gp)


def _assert_layouts_equal(L, m, cfg):
    S, D = L.describe(m, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                      cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    O = oracle.Layout(m, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                      cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    assert O.status == 0
    assert (S.n_ranks, D.n_ranks) == (O.n_src, O.n_dst)
    assert S.n_params == O.n_src_params and D.n_params == O.n_dst_params
    for r in range(S.n_ranks):
        assert S.rank_bytes(r) == O.src_rank_bytes(r), r
        for p in range(S.n_params):
            v = S.param_view(r, p)
            off, r0, r1, c0, c1 = O.src_piece(r, p)
            if r1 <= r0 or c1 <= c0:
                assert v.rows * v.cols == 0, (r, p)
                continue
            assert (v.byte_off, v.full_r0, v.full_r0 + v.rows, v.full_c0, v.full_c0 + v.cols) == \
                (off, r0, r1, c0, c1), (r, p)
    for g in range(D.n_ranks):
        assert D.rank_bytes(g) == O.dst_rank_bytes(g), g
        for gp in range(D.n_params):
            v = D.param_view(g, gp)
            R, C, q, off, soff = O.dst_param(g, gp)
            if R * C == 0:
                assert v.rows * v.cols == 0, (g, gp)
                continue
            assert (v.rows, v.cols, v.quantised, v.byte_off, v.scale_off, v.tensor_scale_off) == \
                (R, C, q, off, soff, O.dst_tensor_scale_off(g, gp)), (g, gp)


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_layout_matches_oracle_full_shapes(L, name):
    """Verdict r1 weak #2: the product's trainer offsets (which its kernels read)
    and generator offsets (which they write) equal the oracle's at the FULL
    benchmark shapes -- the whole model and the slice bench.py times at 1 GPU --
    for every rank and parameter (layout only: cheap)."""
    from paper_2505_24034_b200 import runner
    cfg = CONFIGS[name]
    models = {MODELS[cfg.model], runner.spec_for(name, 1).model()}
    for m in models:
        _assert_layouts_equal(L, m, cfg)


@pytest.mark.parametrize("fsdp,tpt,tpg,dp,sdt,ddt,G", [(4, 1, 1, 4, "f32", "bf16", 8), (2, 2, 2, 3, "bf16", "fp8", 4),
                                                      (3, 1, 4, 2, "f32", "fp8", 2)])
def test_generator_dp_layout_and_plan(L, fsdp, tpt, tpg, dp, sdt, ddt, G):
    m = MODELS["toy"]
    S, D = L.describe(m, fsdp, tpt, tpg, sdt, ddt, dp_gen=dp)
    O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, False, dp)
    assert D.n_ranks == tpg * dp
    for q in range(D.n_ranks):
        assert D.rank_bytes(q) == O.dst_rank_bytes(q)
        for gp in range(D.n_params):
            v = D.param_view(q, gp)
            assert (v.rows, v.cols, v.quantised, v.byte_off, v.scale_off) == O.dst_param(q, gp)
    ns, nd = fsdp * tpt, tpg * dp
    plan = L.Plan(S, D, [r * G // (2 * ns) for r in range(ns)], [G // 2 + q * (G - G // 2) // nd for q in range(nd)])
    src, want = brute.build(m, 8, fsdp, tpt, tpg, sdt, ddt, dp_gen=dp)
    got = _interpret(L, plan, D, src, sdt, ddt, [w.size for w in want])
    for q in range(nd):
        assert np.array_equal(got[q], want[q]), q


@pytest.mark.parametrize("fsdp,tpt,ppt,tpg,ppg,dp,sdt,ddt,G", [
    (2, 1, 2, 2, 1, 1, "f32", "bf16", 4), (1, 2, 1, 2, 2, 1, "bf16", "fp8", 4),
    (3, 1, 2, 4, 2, 2, "f32", "mxfp8", 8), (2, 2, 2, 8, 1, 1, "bf16", "bf16", 8)])
def test_pipeline_stages_layout_and_plan(L, fsdp, tpt, ppt, tpg, ppg, dp, sdt, ddt, G):
    """Decoupled PP (R14): product layouts == oracle's; plan runs == oracle bytes."""
    m = MODELS["toy"]
    S, D = L.describe(m, fsdp, tpt, tpg, sdt, ddt, dp_gen=dp, pp_train=ppt, pp_gen=ppg)
    O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, False, dp, ppt, ppg)
    assert S.n_ranks == O.n_src and D.n_ranks == O.n_dst
    for r in range(S.n_ranks):
        assert S.rank_bytes(r) == O.src_rank_bytes(r)
        for p in range(S.n_params):
            v = S.param_view(r, p)
            off, r0, r1, c0, c1 = O.src_piece(r, p)
            assert v.byte_off == off and v.rows == r1 - r0 and v.cols == c1 - c0
    for q in range(D.n_ranks):
        assert D.rank_bytes(q) == O.dst_rank_bytes(q)
        for gp in range(D.n_params):
            v = D.param_view(q, gp)
            assert (v.rows, v.cols, v.quantised, v.byte_off, v.scale_off) == O.dst_param(q, gp)
    ns, nd = S.n_ranks, D.n_ranks
    plan = L.Plan(S, D, [r * G // ns for r in range(ns)], [q * G // nd for q in range(nd)])
    src, want = brute.build(m, 9, fsdp, tpt, tpg, sdt, ddt, dp_gen=dp, pp_train=ppt, pp_gen=ppg)
    got = _interpret(L, plan, D, src, sdt, ddt, [w.size for w in want])
    for q in range(nd):
        assert np.array_equal(got[q], want[q]), q


@pytest.mark.parametrize("model,fsdp,tpt,tpg,sdt,ddt", [
    ("ragged", 3, 1, 5, "f32", "bf16"), ("ragged", 7, 5, 1, "bf16", "fp8"), ("ragged", 2, 1, 5, "f32", "f32"),
    ("wide", 2, 2, 1, "f32", "bf16"), ("wide", 3, 1, 2, "bf16", "fp8"), ("wide", 1, 2, 1, "f32", "mxfp8"),
    ("head_only", 3, 2, 4, "f32", "bf16"), ("toy", 32, 1, 2, "f32", "bf16")])   # fsdp 32: empty pieces
def test_edge_shapes_plan_runs_reproduce_oracle(L, model, fsdp, tpt, tpg, sdt, ddt):
    m = MODELS[model]
    S, D = L.describe(m, fsdp, tpt, tpg, sdt, ddt)
    plan = L.Plan(S, D, [0] * S.n_ranks, [0] * D.n_ranks)
    src, want = brute.build(m, 31, fsdp, tpt, tpg, sdt, ddt)
    O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt)
    got_o = [np.zeros(O.dst_rank_bytes(g), np.uint8) for g in range(tpg)]
    assert O.sync(src, got_o) == 0
    for a, b in zip(got_o, want):
        assert np.array_equal(a, b)
    got = _interpret(L, plan, D, src, sdt, ddt, [w.size for w in want])
    for g in range(tpg):
        assert np.array_equal(got[g], want[g]), g


def test_mx_rejects_unaligned_shapes(L):
    """MX formats need whole 1x32 row groups inside every tile (R13, R15)."""
    S, D = L.describe(MODELS["ragged"], 1, 1, 5, "f32", "mxfp8")
    with pytest.raises(L.LlrlError) as e:
        L.Plan(S, D, [0], [0] * 5)
    assert e.value.status == L.E_UNSUPPORTED
    with pytest.raises(L.LlrlError) as e:
        L.describe(MODELS["ragged"], 1, 1, 5, "f32", "mxfp4")
    assert e.value.status == L.E_UNSUPPORTED


def test_layout_errors(L):
    m = MODELS["toy"]
    for args, st in [((1, 1, 3), L.E_INDIVISIBLE), ((1, 1, 16), L.E_INDIVISIBLE), ((1, 3, 2), L.E_INDIVISIBLE),
                     ((0, 1, 2), L.E_INVALID)]:
        with pytest.raises(L.LlrlError) as e:
            L.describe(m, *args)
        assert e.value.status == st
    with pytest.raises(L.LlrlError) as e:
        L.describe(m, 1, 1, 2, pp_train=3)        # 2 layers over 3 stages
    assert e.value.status == L.E_INDIVISIBLE
    with pytest.raises(L.LlrlError) as e:
        L.describe(m, 1, 1, 2, "bf16", "f32")
    assert e.value.status == L.E_UNSUPPORTED
    S, _ = L.describe(m, 2, 1, 2)
    _, D2 = L.describe(MODELS["toy"].replace(n_layers=1), 2, 1, 2)
    with pytest.raises(L.LlrlError) as e:
        L.Plan(S, D2, [0, 0], [0, 0])
    assert e.value.status == L.E_MISMATCH


def _interpret(L, plan, D, src_bufs, src_dtype, dst_dtype, dst_sizes):
    """Test-only CPU interpreter of the plan's canonical runs (not a product path)."""
    runs = plan.runs()
    es = {"f32": 4, "bf16": 2}[src_dtype]
    dst = [np.zeros(n, np.uint8) for n in dst_sizes]
    # fp8: assemble generator-local fp32 tensors, then quantise per 128x128 block
    local = {}
    epb = 2 if dst_dtype in ("mxfp4", "nvfp4") else 1          # quantised elements per byte
    for r in runs:
        src = src_bufs[r["src_rank"]]
        raw = src[r["src_off"] * es:(r["src_off"] + r["len"]) * es]
        x = raw.view(np.float32) if src_dtype == "f32" else (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32)
        g = r["dst_rank"]
        if r["flags"] & 1:
            local.setdefault(g, {})
            buf = local[g].setdefault("codes", np.full(dst_sizes[g] * epb, np.nan, np.float32))
            buf[r["dst_off"]:r["dst_off"] + r["len"]] = x
        elif dst_dtype == "f32":
            dst[g][r["dst_off"] * 4:(r["dst_off"] + r["len"]) * 4] = x.view(np.uint8)
        else:
            dst[g][r["dst_off"] * 2:(r["dst_off"] + r["len"]) * 2] = x.astype(ml_dtypes.bfloat16).view(np.uint8)
    for g, d in local.items():
        for gp in range(D.n_params):
            v = D.param_view(g, gp)
            if not v.quantised:
                continue
            e0 = v.byte_off * epb
            x = d["codes"][e0:e0 + v.rows * v.cols].reshape(v.rows, v.cols)
            assert not np.isnan(x).any()
            if dst_dtype == "nvfp4":
                q, s, ts = brute.nv_quant(x)
                dst[g][v.tensor_scale_off:v.tensor_scale_off + 4] = ts.view(np.uint8)
            else:
                quant = {"mxfp8": brute.mx_quant, "mxfp4": brute.mx4_quant}.get(dst_dtype, brute.fp8_quant)
                q, s = quant(x)
            dst[g][v.byte_off:v.byte_off + q.size] = q.reshape(-1)
            dst[g][v.scale_off:v.scale_off + s.nbytes] = s.view(np.uint8).reshape(-1)
    return dst


@pytest.mark.parametrize("fsdp,tpt,tpg,sdt,ddt,inner,G", [
    (2, 1, 2, "f32", "bf16", False, 2),
    (3, 1, 4, "f32", "fp8", False, 2),
    (2, 2, 8, "bf16", "fp8", True, 4),
    (3, 2, 4, "f32", "f32", False, 1),
    (8, 1, 8, "bf16", "bf16", False, 8),
    (2, 4, 8, "bf16", "bf16", False, 8),
    (1, 8, 8, "bf16", "fp8", False, 8),
    (3, 1, 4, "f32", "mxfp8", False, 2),
    (2, 2, 8, "bf16", "mxfp8", True, 4),
    (8, 1, 8, "bf16", "mxfp8", False, 8),
    (3, 1, 4, "f32", "mxfp4", False, 2),
    (2, 2, 8, "bf16", "mxfp4", True, 4),
    (2, 1, 2, "f32", "nvfp4", False, 2),
    (2, 2, 8, "bf16", "nvfp4", True, 4),
])
def test_plan_runs_reproduce_oracle(L, fsdp, tpt, tpg, sdt, ddt, inner, G):
    m = MODELS["toy"]
    S, D = L.describe(m, fsdp, tpt, tpg, sdt, ddt, inner)
    ns, nd = fsdp * tpt, tpg
    plan = L.Plan(S, D, [r * G // ns for r in range(ns)], [g * G // nd for g in range(nd)])
    src, _ = brute.build(m, 4, fsdp, tpt, tpg, sdt, ddt, inner)
    O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, inner)
    want = [np.zeros(O.dst_rank_bytes(g), np.uint8) for g in range(nd)]
    assert O.sync(src, want) == 0
    got = _interpret(L, plan, D, src, sdt, ddt, [w.size for w in want])
    for g in range(nd):
        assert np.array_equal(got[g], want[g]), g


@pytest.mark.parametrize("fsdp,tpt,tpg", [(f, tt, tg) for f in (1, 3, 8) for tt in (1, 2, 8) for tg in (1, 4, 8)])
def test_plan_runs_cover_dst_exactly_once(L, fsdp, tpt, tpg):
    m = MODELS["toy"]
    S, D = L.describe(m, fsdp, tpt, tpg, "f32", "bf16")
    plan = L.Plan(S, D, [0] * (fsdp * tpt), [0] * tpg)
    runs = plan.runs()
    cover = [np.zeros(D.rank_bytes(g) // 2, np.int32) for g in range(tpg)]
    for r in runs:
        cover[r["dst_rank"]][r["dst_off"]:r["dst_off"] + r["len"]] += 1
    for g in range(tpg):
        expect = np.zeros_like(cover[g])
        for gp in range(D.n_params):
            v = D.param_view(g, gp)
            expect[v.byte_off // 2:v.byte_off // 2 + v.rows * v.cols] = 1
        assert np.array_equal(cover[g], expect)


def _plan_for(L, name, G):
    cfg = CONFIGS[name]
    S, D = L.describe(MODELS[cfg.model], cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype,
                      cfg.fsdp_inner)
    sd, dd = placement(cfg, G)
    return L.Plan(S, D, sd, dd)


def test_plan_traffic_matches_survey_appendix_a(L):
    """SURVEY.md App. A "Traffic matrices, G=8 (GB)" [derived] and §8(d) table."""
    t = np.array(_plan_for(L, "c3", 8).traffic()) / 1e9
    assert np.allclose(np.diag(t), 12.354, atol=0.002)
    off = t[~np.eye(8, dtype=bool)]
    assert np.allclose(off, 0.755, atol=0.002)
    t = np.array(_plan_for(L, "c2", 8).traffic()) / 1e9
    for i in range(4):
        assert abs(t[i, 4 + i] - 3.109) < 0.002
        for j in range(4, 8):
            if j != 4 + i:
                assert abs(t[i, j] - 0.302) < 0.002
    assert abs(t.sum() - 16.06) < 0.01
    t = np.array(_plan_for(L, "c5", 8).traffic()) / 1e9
    for i in range(8):   # "10.47 to one peer and 2.28 to another, diagonal local only for GPUs 0 and 7"
        row = sorted(t[i], reverse=True)
        assert abs(row[0] - 10.47) < 0.01 and abs(row[1] - 2.28) < 0.01
        assert (abs(t[i, i] - 10.47) < 0.01) == (i in (0, 7))


def test_plan_bytes_match_baseline_roofline_table(L):
    """BASELINE.md §3 / SURVEY §8(d): C2 at G=1 moves 48.19 GB through HBM;
    C3 at G=8: max HBM/GPU 35.28 GB, max egress 5.29 GB."""
    p = _plan_for(L, "c2", 1)
    b = p.device_bytes(0)
    assert abs((b["hbm_read"] + b["hbm_write"]) / 1e9 - 48.19) < 0.01
    p = _plan_for(L, "c3", 8)
    hbm = max(p.device_bytes(d)["hbm_read"] + p.device_bytes(d)["hbm_write"] for d in range(8)) / 1e9
    tx = max(p.device_bytes(d)["nvl_tx"] for d in range(8)) / 1e9
    assert abs(hbm - 35.28) < 0.01 and abs(tx - 5.29) < 0.01
    s = _plan_for(L, "c4", 8).stats()
    assert s.n_fp8_pull_blocks == 0 and s.n_fp8_blocks == 80 * 52224


def test_c_abi_error_paths(L):
    """No exception or abort crosses the ABI: bad arguments come back as status
    codes with a message (host-only calls; nothing here touches a GPU)."""
    import ctypes
    lib = L.lib()
    m = MODELS["toy"]
    S, D = L.describe(m, 2, 1, 2)
    plan = L.Plan(S, D, [0, 1], [0, 1])
    n = ctypes.c_int64()
    assert lib.llrl_plan_num_runs(None, ctypes.byref(n)) == L.E_INVALID
    assert lib.llrl_layout_rank_bytes(S.handle, 99, ctypes.byref(n)) == L.E_INVALID
    assert b"invalid" in lib.llrl_last_error()
    v = L.ParamView()
    assert lib.llrl_layout_param_view(D.handle, 0, 10 ** 6, ctypes.byref(v)) == L.E_INVALID
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    assert lib.llrl_plan_group_range(plan.handle, 2, 0, 0, ctypes.byref(lo), ctypes.byref(hi)) == L.E_INVALID
    assert lib.llrl_plan_group_range(plan.handle, 0, 0, 99, ctypes.byref(lo), ctypes.byref(hi)) == L.E_INVALID
    # a two-device plan without a comm: llrl_sync refuses before touching CUDA
    ptrs = (ctypes.c_void_p * 2)(1 << 20, 1 << 21)
    assert lib.llrl_sync(plan.handle, None, 0, ptrs, ptrs, None) == L.E_NOPEER
    assert lib.llrl_sync(plan.handle, None, 7, ptrs, ptrs, None) == L.E_INVALID
    # device ordinals out of range, mismatched models
    with pytest.raises(L.LlrlError) as e:
        L.Plan(S, D, [0, 99], [0, 1])
    assert e.value.status == L.E_INVALID
    with pytest.raises(L.LlrlError) as e:
        L.describe(m, 65, 1, 1)            # more than 64 trainer ranks
    assert e.value.status == L.E_INVALID
    # runs: out-of-range requests are errors, in-range ones are exact
    total = plan.num_runs()
    assert plan.runs(total - 1, 1).size == 1
    buf = (L.Run * 2)()
    assert lib.llrl_plan_get_runs(plan.handle, total - 1, 2, buf) == L.E_INVALID


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_plan_algorithmic_bytes_equal_layout_bytes(L, name):
    """The roofline's algorithmic bytes: every byte of every trainer piece is read
    once per generator rank it feeds and every generator byte (data + scales) is
    written once -- checked against the layouts for every benchmark config
    (2-layer versions of the big models)."""
    cfg = CONFIGS[name]
    m = MODELS[cfg.model]
    m = m.replace(n_layers=max(2, cfg.pp_train, cfg.pp_gen)) if m.n_layers > 2 else m
    S, D = L.describe(m, cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype, cfg.fsdp_inner,
                      cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
    sd, dd = placement(cfg, 4)
    plan = L.Plan(S, D, sd, dd)
    st = plan.stats()
    want_dst = 0
    for g in range(D.n_ranks):
        for gp in range(D.n_params):
            v = D.param_view(g, gp)
            n = v.rows * v.cols
            if v.quantised:
                data = n // 2 if cfg.dst_dtype in ("mxfp4", "nvfp4") else n
                if cfg.dst_dtype == "fp8":
                    scales = -(-v.rows // 128) * -(-v.cols // 128) * 4
                elif cfg.dst_dtype == "nvfp4":
                    scales = v.rows * -(-v.cols // 16) + 4        # E4M3 per 1x16 + fp32 tensor scale
                else:
                    scales = v.rows * -(-v.cols // 32)
                want_dst += data + scales
            else:
                want_dst += n * {"f32": 4}.get(cfg.dst_dtype, 2)
    assert st.dst_bytes == want_dst
    want_src = 0                     # every trainer element is read once per generator rank it feeds
    want_reread = 0                  # NVFP4 two-pass: the amax pass reads quantised sources again
    for g in range(D.n_ranks):
        for gp in range(D.n_params):
            v = D.param_view(g, gp)
            n = v.rows * v.cols * {"f32": 4, "bf16": 2}[cfg.src_dtype]
            want_src += n
            want_reread += n if v.quantised and cfg.dst_dtype == "nvfp4" else 0
    assert st.src_bytes == want_src
    dev = [plan.device_bytes(d) for d in range(st.n_devices)]
    assert sum(b["hbm_write"] for b in dev) == st.dst_bytes and sum(b["hbm_read"] for b in dev) == st.src_bytes
    assert sum(plan.device_info(d).nv_amax_read_bytes for d in range(st.n_devices)) == want_reread


def test_nvfp4_group_ranges_include_tensor_scales(L):
    """a layer group's generator byte range covers its NVFP4 tensors'
    fp32 tensor scales (placed after the scale grid), so a caller consuming one
    group at a time gets them."""
    m = MODELS["toy"]
    S, D = L.describe(m, 2, 2, 4, "bf16", "nvfp4")
    plan = L.Plan(S, D, [0] * S.n_ranks, [0] * D.n_ranks)
    n = plan.num_groups()
    for g in range(D.n_ranks):
        for gp in range(D.n_params):
            v = D.param_view(g, gp)
            if not v.quantised:
                continue
            assert v.tensor_scale_off > v.scale_off
            grp = 1 + v.layer                     # groups: embed | layers | final_norm + lm_head
            lo, hi = plan.group_range(1, g, grp)
            assert lo <= v.byte_off and v.tensor_scale_off + 4 <= hi, (g, gp, lo, hi)
    assert n == m.n_layers + 2
