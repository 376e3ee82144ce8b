"""GPU worker (run by test_gpu_parity.test_long_items_claimed_phase in a fresh
process, since LLRL_CHUNK_ELEMS is read once per process): toy syncs whose cast
items span many more shared-memory stages than the ring holds, every item
claimed from the queue (LLRL_STATIC_FRAC=0) and static (=1), through both TMA
cast variants.  The producer then laps the consumers inside an item, so a
consumer that kept reading its item from the recycled hand-off slot (instead of
its own copy) would mix two items.  Prints LONG_OK when every generator byte
equals the oracle's."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import LayoutConfig  # noqa: E402
from tests import harness  # noqa: E402


def main():
    from paper_2505_24034_b200 import runner
    cases = [("f32", "nvfp4", 2, 1, 4), ("f32", "mxfp8", 2, 1, 2), ("bf16", "mxfp4", 1, 1, 1),
             ("f32", "bf16", 3, 1, 4), ("bf16", "bf16", 2, 1, 2)]
    for sdt, ddt, f, tt, tg in cases:
        cfg = LayoutConfig("t", "toy", f, tt, tg, sdt, ddt, "colocated")
        job = runner.SyncJob(runner.JobSpec(cfg, 1), fill=False)
        ol = oracle.Layout(job.model, f, tt, tg, sdt, ddt, False)
        src = harness.host_src(ol, 11)
        for r, t in job.src.items():
            t.copy_(torch.from_numpy(src[r]))
        for g, t in job.dst.items():
            t.fill_(0xA5)
        for _ in range(2):                     # the second sync reuses the queue state
            job.sync()
        torch.cuda.synchronize()
        want = harness.oracle_dst(ol, src, 0xA5)
        for g, t in job.dst.items():
            got = t.cpu().numpy()
            if not np.array_equal(got, want[g]):
                bad = np.nonzero(got != want[g])[0]
                raise SystemExit(f"{sdt}->{ddt} f{f} tt{tt} tg{tg}: dst rank {g}: {bad.size} bytes differ")
        job.close()
    print("LONG_OK", flush=True)


if __name__ == "__main__":
    main()
