"""Host logic of the streamed full-size parity check (tests/harness.py), on CPU
tensors standing in for the GPU buffers: the per-parameter streamed oracle
agrees with the whole-buffer oracle, the partition covers every byte, and
both the value compare and the two-sentinel coverage count catch a wrong or
an unwritten byte."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from synth import MODELS
from tests import harness

CASES = [("toy", 2, 1, 2, "f32", "bf16", 1, 1, 1), ("toy", 3, 2, 4, "bf16", "fp8", 1, 1, 1),
         ("toy", 2, 2, 8, "bf16", "nvfp4", 1, 1, 1), ("toy", 3, 1, 4, "f32", "mxfp4", 2, 1, 1),
         ("toy", 2, 1, 4, "bf16", "mxfp8", 1, 2, 2), ("ragged", 3, 1, 5, "f32", "fp8", 1, 1, 1),
         ("head_only", 2, 1, 2, "f32", "bf16", 1, 1, 1)]


def _layout(model, fsdp, tpt, tpg, sdt, ddt, dp, ppt, ppg):
    ol = oracle.Layout(MODELS[model], fsdp, tpt, tpg, sdt, ddt, False, dp, ppt, ppg)
    assert ol.status == 0
    return ol


@pytest.mark.parametrize("case", CASES)
def test_streamed_compare_matches_whole_oracle(oracle_lib, case):
    ol = _layout(*case)
    seed, s_a, s_b = 7, 0xA5, 0x5A
    src = harness.host_src(ol, seed)
    a = harness.oracle_dst(ol, src, s_a)
    b = harness.oracle_dst(ol, src, s_b)
    dst = {q: torch.from_numpy(a[q].copy()) for q in range(ol.n_dst)}
    n_eq_b = harness.streamed_compare(ol, seed, dst, s_a, count_sentinel=s_b, workers=4)
    for q in range(ol.n_dst):
        parts, pad = harness.dst_partition(ol, q)
        assert parts[0][0] == 0 and parts[-1][1] == a[q].size
        assert all(parts[i][1] == parts[i + 1][0] for i in range(len(parts) - 1))
        assert int(np.count_nonzero(b[q] == s_b)) == n_eq_b[q] + pad
        assert pad == int(np.count_nonzero(a[q] != b[q]))       # the oracle's own padding


def test_streamed_compare_catches_a_wrong_byte(oracle_lib):
    ol = _layout(*CASES[1])
    src = harness.host_src(ol, 3)
    a = harness.oracle_dst(ol, src, 0xA5)
    dst = {q: torch.from_numpy(a[q].copy()) for q in range(ol.n_dst)}
    R, C, q_, off, soff = ol.dst_param(2, 3)
    dst[2][soff + 1] ^= 0x10                       # one byte of an fp8 scale
    with pytest.raises(AssertionError, match="rank 2 param 3"):
        harness.streamed_compare(ol, 3, dst, 0xA5, workers=2)
    dst[2][soff + 1] ^= 0x10
    last = ol.dst_rank_bytes(0) - 1                 # trailing padding written
    dst[0][last] = 0
    with pytest.raises(AssertionError, match="rank 0"):
        harness.streamed_compare(ol, 3, dst, 0xA5, workers=2)


def test_coverage_count_catches_an_unwritten_byte(oracle_lib):
    """A byte the sync never wrote keeps the sentinel of run B, so the count of
    s_b bytes exceeds padding + expected-equal bytes by one."""
    ol = _layout(*CASES[0])
    src = harness.host_src(ol, 5)
    a = harness.oracle_dst(ol, src, 0xA5)
    b = harness.oracle_dst(ol, src, 0x5A)
    off = ol.dst_param(1, 2)[3]
    b[1][off + 3] = 0x5A if a[1][off + 3] != 0x5A else 0x00
    dst = {q: torch.from_numpy(a[q].copy()) for q in range(ol.n_dst)}
    n_eq_b = harness.streamed_compare(ol, 5, dst, 0xA5, count_sentinel=0x5A, workers=2)
    pad = harness.dst_partition(ol, 1)[1]
    assert int(np.count_nonzero(b[1] == 0x5A)) != n_eq_b[1] + pad
