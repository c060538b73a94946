"""Named boundary configurations of BASELINE.json / SURVEY.md §8 (C1-C5).

Each config is an edge (source + destination layouts, batch, width), the
dtypes the boundary carries, and for C4 the placeholder table of the fused
CP-sharded sequence. ``scale`` shrinks the per-sample width for parity tests
while keeping the layouts, which is what the index maps depend on.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .grid import BoundaryEdge, ModuleLayout


@dataclass
class BoundaryConfig:
    name: str
    description: str
    src: ModuleLayout
    dst: ModuleLayout
    batch: int
    tokens: int          # vision tokens per sample (S_v)
    hidden: int          # d_h
    act: str = "bf16"
    grad_in: str = "bf16"
    grad_out: str = "fp32"
    beta: float = 1.0    # backward accumulates into the source-gradient buffer
    splice: dict | None = None  # {"Q", "S", "codes", "text_mode"}
    logical_world: int = 8
    extra: dict = field(default_factory=dict)

    @property
    def width(self) -> int:
        return self.tokens * self.hidden

    def edge(self) -> BoundaryEdge:
        return BoundaryEdge(self.src, self.dst, self.batch, self.width)


def cp_splice_codes(n_images: int, tokens: int, seq_len: int, stride: int, lead: int, seed: int):
    """C4 placeholder table: slot j starts at j*stride+lead and holds image perm[j]."""
    perm = np.random.default_rng(seed).permutation(n_images)
    codes = np.full(seq_len, 0, dtype=np.int64)
    vis = np.zeros(seq_len, dtype=bool)
    for j in range(n_images):
        st = j * stride + lead
        codes[st:st + tokens] = perm[j] * tokens + np.arange(tokens)
        vis[st:st + tokens] = True
    text_idx = np.cumsum(~vis) - 1
    codes[~vis] = -1 - text_idx[~vis]
    return codes.astype(np.int32), perm


def get(name: str, scale: int = 1) -> BoundaryConfig:
    """scale > 1 divides the hidden width (parity runs); layouts are unchanged."""
    name = name.lower()
    h = lambda x: max(8, x // scale)  # noqa: E731
    if name == "c1":
        return BoundaryConfig("c1", "equal-DP enc{dp2} -> llm{dp2}, fp32, 2 simulated ranks",
                              ModuleLayout("encoder", dp=2), ModuleLayout("llm", dp=2), 2, 576,
                              h(4096), act="fp32", grad_in="fp32", grad_out="fp32", logical_world=2)
    if name == "c2":
        return BoundaryConfig("c2", "fan-in colocated vit{dp8} -> llm{tp4,dp2}, bf16 h4096, 64 img x 576",
                              ModuleLayout("vit", dp=8), ModuleLayout("llm", tp=4, dp=2), 64, 576, h(4096))
    if name == "c3":
        return BoundaryConfig("c3", "fan-out colocated enc{tp4,dp2} -> llm{dp8}, bf16 h5120, 64 img x 576",
                              ModuleLayout("encoder", tp=4, dp=2), ModuleLayout("llm", dp=8), 64, 576,
                              h(5120))
    if name == "c4":
        tokens = 576 if scale == 1 else max(4, 576 // scale)
        S = 32768 if scale == 1 else max(32768 // scale, 16 * 2 * tokens)
        S = (S + 63) // 64 * 64
        stride = S // 16
        lead = max(1, stride // 32)
        codes, perm = cp_splice_codes(16, tokens, S, stride, lead, seed=1234)
        return BoundaryConfig("c4", "CP splice vit{dp8} -> llm{tp2,cp4}, S=32768, 16 img x 576 at placeholders",
                              ModuleLayout("vit", dp=8), ModuleLayout("llm", tp=2, cp=4), 16, tokens, h(4096),
                              splice={"Q": 1, "S": S, "codes": codes, "text_mode": 1},
                              extra={"perm": perm.tolist()})
    if name == "c4ip":  # C4 with the in-place splice: the LLM's embedding layer wrote the text rows
        base = get("c4", scale)
        base.name = "c4ip"
        base.description = ("CP splice in place vit{dp8} -> llm{tp2,cp4}, S=32768, 16 img x 576 scattered into "
                            "the LLM's input embeddings at placeholders")
        base.splice = dict(base.splice, text_mode=2)
        return base
    if name == "c5":
        return BoundaryConfig("c5", "non-colocated vit{dp2}@0-1 -> llm{tp2,pp3}@2-7, bf16 h4096, 16 img x 576",
                              ModuleLayout("vit", dp=2), ModuleLayout("llm", tp=2, pp=3, rank_offset=2), 16,
                              576, h(4096))
    # 4-rank variants of the same relations (one process per logical rank on a
    # 4-GPU box; used to exercise the NCCL comparison path and N == world runs).
    if name == "c2w4":
        return BoundaryConfig("c2w4", "fan-in colocated vit{dp4} -> llm{tp2,dp2}, bf16 h4096, 32 img x 576",
                              ModuleLayout("vit", dp=4), ModuleLayout("llm", tp=2, dp=2), 32, 576, h(4096),
                              logical_world=4)
    if name == "c3w4":
        return BoundaryConfig("c3w4", "fan-out colocated enc{tp2,dp2} -> llm{dp4}, bf16 h5120, 32 img x 576",
                              ModuleLayout("encoder", tp=2, dp=2), ModuleLayout("llm", dp=4), 32, 576, h(5120),
                              logical_world=4)
    if name == "c4w4":
        base = get("c4", scale)
        base.name = "c4w4"
        base.description = "CP splice vit{dp4} -> llm{tp2,cp2}, 16 img x 576 at placeholders"
        base.src = ModuleLayout("vit", dp=4)
        base.dst = ModuleLayout("llm", tp=2, cp=2)
        base.logical_world = 4
        return base
    if name == "c5w4":
        return BoundaryConfig("c5w4", "non-colocated vit{dp1}@0 -> llm{tp1,pp3}@1-3, bf16 h4096, 8 img x 576",
                              ModuleLayout("vit", dp=1), ModuleLayout("llm", pp=3, rank_offset=1), 8, 576,
                              h(4096), logical_world=4)
    # 4-GPU stand-ins for the per-GPU traffic of the 8-GPU runs (one rank per
    # GPU, every GPU exchanging with three peers): C2's 4-member all-gather,
    # C3's 4-member gradient gather (diagnostics; N=8 runs only in the driver).
    if name == "c2x4":
        return BoundaryConfig("c2x4", "fan-in colocated vit{dp4} -> llm{tp4}, bf16 h4096, 32 img x 576",
                              ModuleLayout("vit", dp=4), ModuleLayout("llm", tp=4), 32, 576, h(4096),
                              logical_world=4)
    if name == "c3x4":
        return BoundaryConfig("c3x4", "fan-out colocated enc{tp4} -> llm{dp4}, bf16 h5120, 32 img x 576",
                              ModuleLayout("encoder", tp=4), ModuleLayout("llm", dp=4), 32, 576, h(5120),
                              logical_world=4)
    # Deliver layouts: the source's last stage is not the
    # whole rank range, so destination ranks without the data get a DeliverStep.
    if name == "c3p":  # C3' (SURVEY §8 config shorthand): encoder pp4, last stage {r6, r7}
        return BoundaryConfig("c3p", "fan-out with deliver enc{pp4,dp2} -> llm{dp8}, bf16 h5120, 64 img x 576",
                              ModuleLayout("encoder", pp=4, dp=2), ModuleLayout("llm", dp=8), 64, 576, h(5120))
    if name == "appc":  # paper App. C tp2_pp2 colocated doubled: dest stage 0 = {0..3}
        return BoundaryConfig("appc", "equal-DP with deliver vision{tp4,dp2} -> language{tp2,pp2,dp2}, bf16 h4096, "
                                      "64 img x 576",
                              ModuleLayout("vision", tp=4, dp=2), ModuleLayout("language", tp=2, pp=2, dp=2), 64, 576,
                              h(4096))
    raise KeyError(name)


ALL = ["c1", "c2", "c3", "c4", "c5"]


def rank_to_gpu(world: int, n_gpus: int) -> list[int]:
    """logical rank r -> GPU floor(r*N/world) (contiguous blocks)."""
    return [r * n_gpus // world for r in range(world)]
