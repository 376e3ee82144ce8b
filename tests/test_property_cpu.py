"""Property tests (hypothesis) over random model shapes and layouts, CPU only.

For every drawn (model, fsdp, tp_train, tp_gen, dtypes, mesh order, DP
replicas, pipeline stages, GPU count):
* the library's layout validation and the oracle's agree (same accept /
  reject, same error class);
* when valid, the oracle equals the independent brute force (torch.chunk /
  ml_dtypes, tests/brute.py) byte for byte -- a pin of the oracle on shapes no
  hand-written case lists;
* the plan's canonical runs, interpreted on the CPU, reproduce the oracle byte
  for byte, and the runs cover every generator element exactly once.
"""
from __future__ import annotations

import numpy as np
import pytest
from hypothesis import HealthCheck, assume, given, settings, strategies as st

import oracle
from synth.configs import Model
from tests import brute
from tests.test_plan_cpu import _interpret

pytestmark = pytest.mark.filterwarnings("ignore")


@st.composite
def case(draw):
    """Shapes are drawn as multiples of the TP degrees (and, for the MX / NVFP4
    formats, of 32) most of the time, so most draws are valid layouts, with a
    share of arbitrary ones (rejections)."""
    sdt, ddt = draw(st.sampled_from([("f32", "bf16"), ("bf16", "bf16"), ("f32", "f32"), ("bf16", "fp8"),
                                     ("f32", "fp8"), ("bf16", "mxfp8"), ("f32", "mxfp4"), ("bf16", "nvfp4")]))
    tpt = draw(st.sampled_from([1, 2, 3, 4]))
    tpg = draw(st.sampled_from([1, 2, 3, 4, 6, 8]))
    lcm = tpt * tpg // np.gcd(tpt, tpg)
    unit = lcm if draw(st.integers(0, 4)) else 1
    if ddt in ("mxfp8", "mxfp4", "nvfp4") and draw(st.integers(0, 3)):
        unit *= 32                                    # whole 1x32 / 1x16 row groups per shard
    hd = draw(st.sampled_from([4, 8, 16, 32]))
    kv = draw(st.sampled_from(sorted({1, 2, 3, 4, tpg})))
    heads = kv * draw(st.sampled_from(sorted({1, 2, 3, lcm})))
    m = Model(draw(st.integers(0, 2)), unit * draw(st.sampled_from([1, 2, 3])) * 8, heads, kv, hd,
              unit * draw(st.sampled_from([8, 12, 20, 32])), unit * draw(st.sampled_from([4, 6, 8, 10])),
              draw(st.integers(0, 1)))
    if m.n_layers == 0:
        m = m.replace(with_embed=1)
    d, q, k = m.d_model, m.n_heads * m.head_dim, m.n_kv_heads * m.head_dim
    n_el = m.n_layers * (d * (q + 2 * k) + q * d + 3 * d * m.d_ffn) + 2 * m.vocab * d * m.with_embed
    assume(n_el <= 600_000)                           # keep each example well under a second
    fsdp = draw(st.integers(1, 5))
    inner = draw(st.booleans())
    dp = draw(st.sampled_from([1, 1, 2]))
    ppt = draw(st.sampled_from([1, 1, 2]))
    ppg = draw(st.sampled_from([1, 1, 2]))
    G = draw(st.integers(1, 4))
    return m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg, G


@settings(max_examples=200, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(case())
def test_random_layouts_plan_and_oracle(c):
    from paper_2505_24034_b200 import llrl as L
    m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg, G = c
    O = oracle.Layout(m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg)
    try:
        S, D = L.describe(m, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg)
    except L.LlrlError as e:
        assert O.status != 0, f"library rejects ({e}), oracle accepts {c}"
        assert O.status == e.status, (O.status, e.status, c)
        return
    assert O.status == 0, f"oracle rejects ({O.status}), library accepts {c}"
    ns, nd = fsdp * tpt * ppt, tpg * ppg * dp
    assert (S.n_ranks, D.n_ranks) == (ns, nd)
    src, want_brute = brute.build(m, 5, fsdp, tpt, tpg, sdt, ddt, inner, dp, ppt, ppg)
    want = [np.zeros(O.dst_rank_bytes(g), np.uint8) for g in range(nd)]
    assert O.sync(src, want) == 0
    for g in range(nd):
        assert np.array_equal(want[g][:want_brute[g].size], want_brute[g]), (g, c)
    try:
        plan = L.Plan(S, D, [r * G // ns for r in range(ns)], [g * G // nd for g in range(nd)])
    except L.LlrlError as e:
        # R13 / R15 / R16: tiles that split a 1x32 (1x16) row group are UNSUPPORTED
        # (the oracle defines partial groups; the kernels quantise whole groups)
        assert ddt in ("mxfp8", "mxfp4", "nvfp4") and e.status == L.E_UNSUPPORTED, (e, c)
        return
    got = _interpret(L, plan, D, src, sdt, ddt, [w.size for w in want])
    for g in range(nd):
        assert np.array_equal(got[g], want[g]), (g, c)
    # exactly-once coverage of every generator element by the runs
    cover = [np.zeros(2 * D.rank_bytes(g), np.int32) for g in range(nd)]   # in half-bytes
    fp4 = ddt in ("mxfp4", "nvfp4")
    for r in plan.runs():
        g, o, n = r["dst_rank"], r["dst_off"], r["len"]
        # nibbles per element: f32 8, bf16 4; quantised (flag 1) codes: fp8 / MXFP8 2, fp4 1
        h = 8 if ddt == "f32" else (1 if fp4 else 2) if r["flags"] & 1 else 4
        cover[g][o * h:(o + n) * h] += 1
    for g in range(nd):
        assert cover[g].max() <= 1, (g, c)
    plan.close()
