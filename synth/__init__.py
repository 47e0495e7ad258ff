"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module only *constructs inputs*: it draws seeded Gaussians, plants row- or
column-wise outliers and rounds to bf16 so that the oracle and the CUDA path see
the very same buffer. It holds none of the method's arithmetic (no Hadamard, no
quantiser, no top-k, no GEMM) and imports neither ``oracle`` nor the product
package.

Recipe:
  * RNG: numpy ``Generator(Philox(key))`` with key = 42 + case id (SPEC S:560
    default seed 42; counter-based generator per S:409). The torch variant used
    for full-size bench inputs draws with ``torch.Generator(device).manual_seed``.
  * base distributions: X ~ N(0,1), W ~ N(0, 0.02^2), G_Y ~ N(0, 1e-3^2)
  * planting in the FED orientation (rows/cols of the tensor as given):
      R: ceil(0.1% * rows) (min 1) rows scaled by 100
      C: ceil(0.1% * cols) (min 1) columns scaled by 100
      N: nothing planted
  * values rounded RNE to bf16 (returned as float32 arrays holding bf16 values)
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SIGMA = {"X": 1.0, "W": 0.02, "GY": 1e-3}
PLANT_SCALE = 100.0
PLANT_FRACTION = 0.001


def rng(case_id: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=42 + int(case_id)))


def n_planted(dim: int) -> int:
    return max(1, math.ceil(PLANT_FRACTION * dim))


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def to_bf16_bits(x_bf16_valued: np.ndarray) -> np.ndarray:
    """float32 array holding bf16 values -> uint16 bf16 bit patterns (exact)."""
    x = np.ascontiguousarray(x_bf16_valued, dtype=np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)


@dataclass
class Planted:
    rows: np.ndarray  # planted row indices (fed orientation)
    cols: np.ndarray  # planted column indices


def operand(rows: int, cols: int, pattern: str, kind: str = "X", case_id: int = 0,
            scale: float = PLANT_SCALE, count: int | None = None, bf16: bool = True):
    """One seeded operand of shape rows x cols with `pattern` in {'R','C','N'}.

    Returns (array float32, Planted). The pattern refers to the tensor exactly as
    returned (its fed orientation when it is passed as a GEMM operand)."""
    g = rng(case_id)
    a = g.standard_normal((rows, cols), dtype=np.float32) * np.float32(SIGMA[kind])
    pr = np.zeros(0, np.int64)
    pc = np.zeros(0, np.int64)
    if pattern == "R":
        c = count if count is not None else n_planted(rows)
        pr = np.sort(g.choice(rows, size=c, replace=False))
        a[pr, :] *= np.float32(scale)
    elif pattern == "C":
        c = count if count is not None else n_planted(cols)
        pc = np.sort(g.choice(cols, size=c, replace=False))
        a[:, pc] *= np.float32(scale)
    elif pattern != "N":
        raise ValueError(pattern)
    if bf16:
        a = round_bf16(a)
    return a, Planted(pr, pc)


def operand_torch(rows: int, cols: int, pattern: str, kind: str, seed: int, device,
                  scale: float = PLANT_SCALE, plant_seed: int | None = None, out=None):
    """Full-size bench operand generated on the device (bf16), same recipe. With plant_seed the
    planted rows / columns come from their own generator, so that successive steps (different
    `seed`) keep the same outlier channels — the persistence calibration relies on.
    `out` (bf16, rows x cols) receives the result in place."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(42 + int(seed))
    a = torch.randn((rows, cols), generator=g, device=device, dtype=torch.float32)
    a.mul_(SIGMA[kind])
    gp = g
    if plant_seed is not None:
        gp = torch.Generator(device=device)
        gp.manual_seed(42 + int(plant_seed))
    if pattern == "R":
        idx = torch.randperm(rows, generator=gp, device=device)[: n_planted(rows)]
        a[idx, :] *= scale
    elif pattern == "C":
        idx = torch.randperm(cols, generator=gp, device=device)[: n_planted(cols)]
        a[:, idx] *= scale
    if out is not None:
        return out.copy_(a)
    return a.to(torch.bfloat16)


# Config 5: per-tensor patterns of the 16 x 7 Llama-3.2-1B linears that reproduce the
# model's Table-1 census exactly: 15 linears (X = N, G_Y = C), 69 (C, C), 20 (C, N),
# 8 (C, R) placed on k / v projections; W = N everywhere.
def llama32_1b_census_patterns():
    """[(layer, linear, pattern_x, pattern_w, pattern_gy)] for the 112 linears."""
    names = [n for n, _, _ in LLAMA32_1B["linears"]]
    slots = [(layer, n) for layer in range(LLAMA32_1B["layers"]) for n in names]
    kv = [s for s in slots if s[1] in ("k", "v")][:8]
    rest = [s for s in slots if s not in kv]
    cls = {s: ("C", "R") for s in kv}
    for i, s in enumerate(rest):
        cls[s] = ("N", "C") if i < 15 else (("C", "C") if i < 15 + 69 else ("C", "N"))
    return [(layer, n, cls[(layer, n)][0], "N", cls[(layer, n)][1]) for layer, n in slots]


# --------------------------------------------------------------------------------------
# Workload shapes (BASELINE.json configs)
# --------------------------------------------------------------------------------------
# Llama-3.2-1B: hidden 2048, MLP 8192, kv 512 (8 kv heads x 64); T = seq 2048 x batch 8.
LLAMA32_1B = {
    "hidden": 2048, "mlp": 8192, "kv": 512, "layers": 16, "tokens": 16384,
    # (name, d_in, d_out)
    "linears": [("q", 2048, 2048), ("k", 2048, 512), ("v", 2048, 512), ("o", 2048, 2048),
                ("gate", 2048, 8192), ("up", 2048, 8192), ("down", 8192, 2048)],
}
LLAMA3_8B = {
    "hidden": 4096, "mlp": 14336, "kv": 1024, "layers": 32, "tokens": 16384,
    "linears": [("q", 4096, 4096), ("k", 4096, 1024), ("v", 4096, 1024), ("o", 4096, 4096),
                ("gate", 4096, 14336), ("up", 4096, 14336), ("down", 14336, 4096)],
}
# Instella-3B (BASELINE configs[2]): 36 layers (Table 1: 252 linears / 7), hidden 2560, MLP 6912,
# multi-head attention (k / v as wide as q) — the public model card's shapes, no weights needed.
INSTELLA_3B = {
    "hidden": 2560, "mlp": 6912, "kv": 2560, "layers": 36, "tokens": 16384,
    "linears": [("q", 2560, 2560), ("k", 2560, 2560), ("v", 2560, 2560), ("o", 2560, 2560),
                ("gate", 2560, 6912), ("up", 2560, 6912), ("down", 6912, 2560)],
}

# Per-linear tensor patterns for one Llama-3.2-1B layer used by the bench step. They are
# drawn from the Table-1 census classes: X is C or N,
# W is always N, G_Y is C, N or R. (X, G_Y) per linear:
LLAMA32_1B_LAYER_PATTERNS = {
    "q": ("C", "C"), "k": ("C", "R"), "v": ("C", "C"), "o": ("N", "C"),
    "gate": ("C", "C"), "up": ("C", "N"), "down": ("C", "C"),
}
