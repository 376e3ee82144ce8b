#!/usr/bin/env python
"""Per-CTA timeline of the cast launch (verdict r1 #8: where does the tail of an
NVLink-bound sync come from?).  Runs one config like bench.py, with
LLRL_TIMELINE=1, and prints per GPU the CTA start / end spread:

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
      tools/timeline.py --config c3 --gpus 4
"""
from __future__ import annotations

import argparse
import json
import os
import sys

os.environ["LLRL_TIMELINE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2505_24034_b200 import runner
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    job = runner.SyncJob(runner.spec_for(args.config, args.gpus), device=local, seed=0)
    out = []
    for rep in range(args.reps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        job.sync()
        torch.cuda.synchronize()
        tl = job.plan.debug_timeline(job.device)
        if not tl:
            continue
        t0 = min(s for s, _ in tl)
        ends = sorted((e - t0) / 1e6 for _, e in tl)
        starts = sorted((s - t0) / 1e6 for s, _ in tl)
        n = len(ends)
        out.append({"rep": rep, "gpu": job.device, "ctas": n, "start_max_ms": round(starts[-1], 4),
                    "end_min_ms": round(ends[0], 4), "end_p10_ms": round(ends[n // 10], 4),
                    "end_p50_ms": round(ends[n // 2], 4), "end_p90_ms": round(ends[9 * n // 10], 4),
                    "end_max_ms": round(ends[-1], 4)})
    allo = [None] * world
    if world > 1:
        dist.all_gather_object(allo, out)
    else:
        allo = [out]
    if job.rank == 0:
        for o in allo:
            for r in o:
                print(json.dumps(r))
    job.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
