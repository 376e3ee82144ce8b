"""bench.py contract checks that need no GPU: the reference arm (the CPU
oracle, `--impl reference`) prints one JSON line with the contract's keys, and
our arm refuses to run without CUDA (no CPU fallback)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "ms" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"] and "model" not in d["config"]


def test_our_arm_fails_without_cuda():
    import torch
    if torch.cuda.is_available():
        return
    r = _run(["--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"])
    assert r.returncode != 0
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")], "printed a number without a GPU"


def test_reference_arm_whole_workload_and_same_config():
    """The reference arm times the whole workload each step (no extrapolation),
    parameter-parallel over every host core, and reports the same `config`
    object as our arm (bench.config_dict of the same arguments)."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    from synth import CONFIGS
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3"])
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    args = argparse.Namespace(gpus=1, max_ctas=0, multicast=False, replicate="push", step_sync=False,
                              placement=None)
    cfg = CONFIGS["c1"]
    assert d["config"] == bench.config_dict(cfg, args, bench._model_for(cfg, 1))
    cb = d["cpu_baseline"]
    assert cb["cores"] == os.cpu_count() and "no extrapolation" in cb["sample"]
    assert "extrapolat" not in cb["sample"].replace("no extrapolation", "")


def test_cpu_baseline_times_the_whole_workload():
    sys.path.insert(0, ROOT)
    import bench
    from synth import CONFIGS
    out = bench.cpu_baseline(CONFIGS["c1"], 1)
    assert out["cores"] == os.cpu_count() and out["value"] > 0 and out["single_thread_ms"] > 0
    assert out["nproc"] == os.cpu_count() and out["cpu_model"]


def _expand(R):
    """rectangles back to sorted (src_rank, dst_rank, src_off, dst_off, len) runs"""
    import numpy as np
    sr, dr, so, do, ln, rows, ss, ds = R
    k = np.repeat(np.arange(len(sr)), rows)
    j = np.arange(len(k)) - np.repeat(np.cumsum(rows) - rows, rows)
    out = np.stack([sr[k], dr[k], so[k] + j * ss[k], do[k] + j * ds[k], ln[k]], 1)
    return out[np.lexsort(out.T[::-1])]


def test_ce_comparator_rectangles_cover_the_runs():
    """bench.py's copy-engine comparator copies exactly the plan's runs: its 2-D
    rectangles expand back to the runs (toy sweep and C5 at 4 GPUs), and the
    strided o / down tiles coalesce (far fewer copies than runs)."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from paper_2505_24034_b200 import llrl, runner
    from synth.configs import placement
    for name, n in (("c1", 1), ("c3", 4), ("c5", 4), ("c8", 4)):
        spec = runner.spec_for(name, n)
        cfg = spec.cfg
        if name != "c1":
            spec = runner.JobSpec(cfg, n, n_layers=2)
        S, D = llrl.describe(spec.model(), cfg.fsdp, cfg.tp_train, cfg.tp_gen, cfg.src_dtype, cfg.dst_dtype,
                             cfg.fsdp_inner, cfg.dp_gen, cfg.pp_train, cfg.pp_gen)
        sd, dd = placement(cfg, n)
        P = llrl.Plan(S, D, sd, dd)
        runs = P.runs()
        R = bench._rectangles(runs)
        want = np.stack([runs["src_rank"], runs["dst_rank"], runs["src_off"], runs["dst_off"], runs["len"]], 1)
        want = want[np.lexsort(want.T[::-1])]
        assert np.array_equal(_expand(R), want), name
        assert (R[6] >= R[4]).all() and (R[7] >= R[4]).all()      # forward 2-D patterns
        if name != "c1":
            assert len(R[0]) * 100 < len(runs), (name, len(R[0]), len(runs))
        P.close()
