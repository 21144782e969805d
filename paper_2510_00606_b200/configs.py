"""Model-state geometries of the BASELINE.json configurations.

Layer-size vectors follow SURVEY Appendix A ("Layer-size vectors used for the
config probes"): bytes = params x bytes/param, one entry per ZeroLayout layer.
All state is synthetic (no checkpoints exist offline): word i of the flat
space is splitmix64(seed ^ i).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class StateConfig:
    name: str
    layer_params: List[int]
    bytes_per_param: int
    dp: int

    @property
    def layer_bytes(self) -> List[int]:
        return [p * self.bytes_per_param for p in self.layer_params]

    @property
    def total_bytes(self) -> int:
        return sum(self.layer_bytes)

    @property
    def params(self) -> int:
        return sum(self.layer_params)


def gpt_125m() -> StateConfig:
    """Config A: 123.65 M params, fp32 param + Adam m, v (12 B/param), DP=4."""
    return StateConfig("125M-fp32-adam", [38_597_376] + [7_087_872] * 12, 12, 4)


def llama2_7b() -> StateConfig:
    """Config B: 6,738,415,616 params, bf16 param + fp32 master/m/v (14 B), DP=8."""
    return StateConfig("llama2-7b-zero", [131_072_000] + [202_383_360] * 32 + [131_076_096],
                       14, 8)


def llama2_7b_per_tensor() -> StateConfig:
    """Config B at per-tensor granularity (291 tensors)."""
    h, f = 4096, 11008
    layers = [131_072_000]
    for _ in range(32):
        layers += [h * h] * 4 + [h * f] * 3 + [h, h]
    layers += [h, 131_072_000]
    return StateConfig("llama2-7b-zero-per-tensor", layers, 14, 8)


def llama3_8b() -> StateConfig:
    """Config C: 8,030,261,248 params x 14 B, DP=8 (8 -> 6 -> 8)."""
    return StateConfig("llama3-8b-zero", [525_336_576] + [218_112_000] * 32 + [525_340_672],
                       14, 8)


def fill_hbm(n_gpus: int, per_gpu_bytes: int = 88_000_000_000) -> StateConfig:
    """Config D: ZeRO state sized to fill ~180 GB HBM per GPU (80 layers)."""
    total = per_gpu_bytes * n_gpus
    return StateConfig(f"fill-hbm-{n_gpus}", [total // 80] * 80, 1, n_gpus)


def scaled(cfg: StateConfig, factor: float, name_suffix: str = "") -> StateConfig:
    """Same layer structure, every layer scaled (parity tests at small size)."""
    return StateConfig(cfg.name + (name_suffix or f"-x{factor:g}"),
                       [max(1, int(p * factor)) for p in cfg.layer_params],
                       cfg.bytes_per_param, cfg.dp)
