"""Benchmark workloads of BASELINE.json (configs A-E).

Masks come from the reference generator restated bit-exactly in the product
(generate_mask_set, pinned by tests/test_planner_golden.py); Q/K/V are
synthetic bf16 N(0,1) from one fixed seed, global [S, H, d], sharded by token
blocks.  Block size is 64 everywhere.
"""
from __future__ import annotations

from dataclasses import dataclass

from .planner import GeneratorSpec


@dataclass(frozen=True)
class Workload:
    name: str
    heads: int
    head_dim: int
    tokens: int
    pattern: str
    min_density: float
    max_density: float
    seed: int = 1
    gpus_hint: int = 8
    note: str = ""

    @property
    def blocks(self) -> int:
        return -(-self.tokens // 64)

    def spec(self, seed: int = None) -> GeneratorSpec:
        return GeneratorSpec(self.heads, self.blocks, self.blocks, 64, self.pattern, self.min_density,
                             self.max_density, 1.0, self.seed if seed is None else seed)

    def flops_per_block(self) -> int:
        # QK^T + PV on one dense 64x64 tile: 2 * (2 * 64 * 64 * d)
        return 4 * 64 * 64 * self.head_dim

    def describe(self) -> dict:
        return {"workload": self.name, "heads": self.heads, "head_dim": self.head_dim,
                "tokens": self.tokens, "block": 64, "mask": self.pattern,
                "density_ramp": [self.min_density, self.max_density], "mask_seed": self.seed}


WORKLOADS = {
    # A: CPU-ref toy (BASELINE configs[0]).
    "toy": Workload("toy-A", 8, 64, 4096, "random", 0.5, 0.5, 1, 4,
                    "8 heads, 4096 tokens, d=64, 50% random, simulated SP=4 (U2R2)"),
    # B: CogVideoX-5B-shaped layer (configs[1]); PARO mean density 0.317
    # with a per-head ramp 0.15-0.484: real PARO/Sparge masks
    # differ per head (the reference reports rho_s 1.45 for Ulysses on
    # CogVideoX1.5), a constant density would hide that.
    "cogvideox": Workload("cogvideox-5b-B", 48, 64, 17792, "clustered", 0.15, 0.484, 1, 8,
                          "48 heads, d=64, 278 blocks, clustered ramp 0.15-0.484 (mean 0.317)"),
    "cogvideox-flat": Workload("cogvideox-5b-B-flat", 48, 64, 17792, "clustered", 0.317, 0.317, 1, 8,
                               "48 heads, d=64, 278 blocks, every head at density 0.317"),
    # C: Wan2.1-T2V-14B 480p layer (configs[2]) -- the north-star workload.
    "wan": Workload("wan2.1-14b-480p-C", 40, 128, 32768, "clustered", 0.15, 0.45, 1, 8,
                    "40 heads, d=128, 512 blocks, clustered 0.15-0.45 (mean 0.30)"),
    # C with the other two generator families (report all
    # three; uniform splits are already near-balanced on these).
    "wan-random": Workload("wan2.1-14b-480p-C-random", 40, 128, 32768, "random", 0.15, 0.45, 1, 8,
                           "as C, uniform Bernoulli masks 0.15-0.45"),
    "wan-banded": Workload("wan2.1-14b-480p-C-banded", 40, 128, 32768, "banded", 0.15, 0.45, 1, 8,
                           "as C, banded masks 0.15-0.45"),
    # D: HunyuanVideo 720p layer (configs[3]).
    "hunyuan": Workload("hunyuanvideo-720p-D", 24, 128, 118848, "clustered", 0.15, 0.45, 1, 8,
                        "24 heads, d=128, 1857 blocks, ~30% density"),
}
