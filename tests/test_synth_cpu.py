"""The C twin of the input generator (synth/synth.c) gives the same bits as the
numpy definition (synth.weight_bits) -- the full-size GPU parity tests and
bench.py's CPU legs fill their trainer buffers with it."""
from __future__ import annotations

import numpy as np
import pytest

import synth
from synth import fast


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("is_norm", [False, True])
def test_c_generator_matches_numpy(dtype, is_norm):
    rng = np.random.default_rng(0)
    for seed, param in ((0, 0), (1, 17), (11, 722), (2 ** 40 + 3, 5)):
        r0, c0 = int(rng.integers(0, 1 << 17)), int(rng.integers(0, 1 << 15))
        nr, nc = 37, 301
        want = synth.weight_bits(seed, param, is_norm, dtype, np.arange(r0, r0 + nr)[:, None],
                                 np.arange(c0, c0 + nc)[None, :])
        got = fast.weight_bits(seed, param, is_norm, dtype, r0, r0 + nr, c0, c0 + nc)
        assert got.dtype == want.dtype and np.array_equal(got, want)


def test_c_generator_threaded_matches_single():
    """The row-split multi-threaded fill equals one single-threaded call."""
    a = np.empty((3000, 700), np.uint32)
    b = np.empty_like(a)
    fast.fill(a, 4, 9, False, "f32", 100, 3100, 3, 703, parallel=True)
    fast.fill(b, 4, 9, False, "f32", 100, 3100, 3, 703, parallel=False)
    assert np.array_equal(a, b)
    assert np.array_equal(a[1234:1240], synth.weight_bits(4, 9, False, "f32", np.arange(1334, 1340)[:, None],
                                                          np.arange(3, 703)[None, :]))
