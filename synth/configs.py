"""Model shapes and layout configurations of the benchmark workloads.

Shapes: Llama-3.1 config.json values [ext]; PAPER.md names the models only
("LLaMA 3.1" 8B / 70B / 405B).  Layout configurations C1-C5 are
BASELINE.json ``configs`` [0..4] (SURVEY.md §8 "Per-rank buffers").
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict


@dataclass(frozen=True)
class Model:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ffn: int
    vocab: int
    with_embed: int = 1

    def replace(self, **kw) -> "Model":
        d = asdict(self)
        d.update(kw)
        return Model(**d)


MODELS = {
    "toy": Model(2, 256, 8, 2, 32, 1024, 512, 1),
    # edge-case shapes for parity tests: "ragged" (no dimension a multiple of 8:
    # scalar fallbacks, partial fp8 blocks), "wide" (rows wider than a 32 KiB TMA
    # stage: column-segmented chunks), "head_only" (no decoder layer)
    "ragged": Model(1, 20, 5, 5, 4, 30, 10, 1),
    "wide": Model(1, 64, 2, 1, 32, 20480, 64, 1),
    "head_only": Model(0, 256, 8, 2, 32, 1024, 512, 1),
    "llama3-8b": Model(32, 4096, 32, 8, 128, 14336, 128256, 1),
    "llama3-70b": Model(80, 8192, 64, 8, 128, 28672, 128256, 1),
    "llama3-405b": Model(126, 16384, 128, 8, 128, 53248, 128256, 1),
    "llama3-405b-slice16": Model(16, 16384, 128, 8, 128, 53248, 128256, 0),
}


@dataclass(frozen=True)
class LayoutConfig:
    """One trainer->generator layout pair."""
    name: str
    model: str
    fsdp: int
    tp_train: int
    tp_gen: int
    src_dtype: str          # "f32" | "bf16"
    dst_dtype: str          # "f32" | "bf16" | "fp8"
    placement: str          # "disjoint" | "colocated" | "rotated" | "fanout"
    fsdp_inner: bool = False
    notes: str = ""
    dp_gen: int = 1         # generator data-parallel replicas (R12)
    pp_train: int = 1       # pipeline stages (R14)
    pp_gen: int = 1

    @property
    def n_src(self) -> int:
        return self.fsdp * self.tp_train * self.pp_train

    @property
    def n_dst(self) -> int:
        return self.tp_gen * self.pp_gen * self.dp_gen


CONFIGS = {
    "c1": LayoutConfig("c1", "toy", 2, 1, 2, "f32", "bf16", "disjoint",
                       notes="toy fp32 FSDP=2 -> bf16 TP=2"),
    "c2": LayoutConfig("c2", "llama3-8b", 4, 1, 4, "f32", "bf16", "disjoint",
                       notes="8B fp32 FSDP=4 (GPUs 0..G/2) -> bf16 TP=4 (GPUs G/2..G)"),
    "c3": LayoutConfig("c3", "llama3-70b", 8, 1, 8, "bf16", "bf16", "colocated",
                       notes="70B bf16 FSDP=8 -> bf16 TP=8, co-located"),
    "c4": LayoutConfig("c4", "llama3-70b", 1, 8, 8, "bf16", "fp8", "colocated",
                       notes="70B bf16 TP=8 -> fp8 TP=8 with 128x128 block scales"),
    "c5": LayoutConfig("c5", "llama3-405b-slice16", 2, 4, 8, "bf16", "bf16", "colocated",
                       notes="405B 16-layer slice FSDP=2xTP=4 -> TP=8, TP-innermost mesh"),
    # NEXT f1: a generator pool of DP replicas, here the
    # paper's best 8B setting "gen mp 1" with 4 replicas fed by a 4-GPU trainer.
    "c6": LayoutConfig("c6", "llama3-8b", 4, 1, 1, "bf16", "bf16", "disjoint", dp_gen=4,
                       notes="8B bf16 FSDP=4 (GPUs 0..G/2) -> bf16 TP=1 x DP=4 replicas (GPUs G/2..G)"),
    # NEXT f2: MX formats for the generator, as tcgen05 block-scaled MMA consumes them
    "c7": LayoutConfig("c7", "llama3-70b", 1, 8, 8, "bf16", "mxfp8", "colocated",
                       notes="70B bf16 TP=8 -> MXFP8 TP=8 (E4M3 + E8M0 per 1x32)"),
    "c10": LayoutConfig("c10", "llama3-70b", 1, 8, 8, "bf16", "mxfp4", "colocated",
                        notes="70B bf16 TP=8 -> MXFP4 TP=8 (E2M1 + E8M0 per 1x32)"),
    "c11": LayoutConfig("c11", "llama3-70b", 1, 8, 8, "bf16", "nvfp4", "colocated",
                        notes="70B bf16 TP=8 -> NVFP4 TP=8 (E2M1 + E4M3 per 1x16 + fp32 per tensor)"),
    # NVFP4 with the per-tensor amax reduced across GPUs: FSDP=8 chunks of every
    # generator tensor sit on several GPUs (the cross-GPU handshake of R16)
    "c12": LayoutConfig("c12", "llama3-70b", 8, 1, 8, "bf16", "nvfp4", "colocated",
                        notes="70B bf16 FSDP=8 -> NVFP4 TP=8 (cross-GPU tensor amax)"),
    # NEXT f1 with NVLS multicast: more generator replicas than trainer GPUs, so the
    # trainer's NVLink egress binds without multicast (3 copies) and not with it (1 copy).
    "c9": LayoutConfig("c9", "llama3-8b", 1, 1, 1, "bf16", "bf16", "fanout", dp_gen=3,
                       notes="8B bf16 trainer on GPU 0 -> 3 bf16 TP=1 DP replicas on GPUs 1..3 (multicast fan-out)"),
    # NEXT f4: decoupled pipeline parallelism -- a PP=2 trainer
    # (FSDP=2 x TP=2 per stage) re-staged into a PP-less TP=8 generator.
    "c8": LayoutConfig("c8", "llama3-70b", 2, 2, 8, "bf16", "bf16", "colocated", pp_train=2,
                       notes="70B bf16 PP=2 x FSDP=2 x TP=2 -> bf16 TP=8 (layer re-staging)"),
}


def placement(cfg: LayoutConfig, n_gpus: int):
    """Logical rank -> GPU ordinal maps (src_device[], dst_device[]).

    SURVEY.md §8(d) "Placements": C2 uses disjoint halves for G >= 2 (trainer
    ranks block-mapped onto GPUs [0, G/2), generator onto [G/2, G)) and all on
    GPU 0 at G = 1; co-located configs map logical rank r -> GPU floor(r*G/n)
    on both sides; "rotated" shifts the trainer by one GPU.
    """
    ns, nd = cfg.n_src, cfg.n_dst
    if n_gpus == 1:
        return [0] * ns, [0] * nd
    if cfg.placement == "fanout":          # trainer on GPU 0, generator ranks over GPUs 1..G-1
        return [0] * ns, [1 + g * (n_gpus - 1) // nd for g in range(nd)]
    if cfg.placement == "disjoint":
        half = n_gpus // 2
        return ([r * half // ns for r in range(ns)],
                [half + g * (n_gpus - half) // nd for g in range(nd)])
    src = [r * n_gpus // ns for r in range(ns)]
    dst = [g * n_gpus // nd for g in range(nd)]
    if cfg.placement == "rotated":
        src = [(d + 1) % n_gpus for d in src]
    return src, dst
