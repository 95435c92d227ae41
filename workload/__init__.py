"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws matrices and
sample positions.  Both the oracle (``oracle/``) and the CUDA path
(``paper_1106_1347_b200``) consume what it produces; neither is imported here.

Recipe:
  * generator: numpy PCG64 seeded by SeedSequence([11061347, cfg, mat, variant, chunk]),
    mat 0 = A, 1 = B; variant 0 = real, 1 = integer-valued; chunk = 1024-row block,
    so any row range (a rank's shard) regenerates independently of the world size.
  * BASELINE.json configs:
      c1 N=P=M=128     real U[-1,1)        int {-8..8}
      c2 N=P=M=1024    real U[-1,1)        int {-8..8}
      c3 4096x1001x3000  A = U[-1,1)*1e6, B = U[-1,1)*1e-6 (ill-scaled, odd P)
      c4 N=P=M=8192    standard normal
      c5 N=P=M=32768   real U[-1,1)
  * paper protocol: A ~ U[0,1) n x n, B = 8A (exact).
  * sample positions: SeedSequence([11061347, cfg, 99, shard]).
The paper measures on no public dataset; these synthetic matrices are the whole workload.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

SEED = 11061347
CHUNK = 1024


@dataclass(frozen=True)
class Config:
    key: str
    cfg_id: int
    N: int
    P: int
    M: int
    dist: str  # "uniform" | "scaled" | "normal"
    has_int: bool

    @property
    def flops(self) -> float:
        return 2.0 * self.N * self.P * self.M


CONFIGS = {
    "c1": Config("c1", 1, 128, 128, 128, "uniform", True),
    "c2": Config("c2", 2, 1024, 1024, 1024, "uniform", True),
    "c3": Config("c3", 3, 4096, 1001, 3000, "scaled", False),
    "c4": Config("c4", 4, 8192, 8192, 8192, "normal", False),
    "c5": Config("c5", 5, 32768, 32768, 32768, "uniform", False),
}


def _chunk_rng(cfg_id: int, mat: int, variant: int, chunk: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED, cfg_id, mat, variant, chunk])))


def _draw(rng: np.random.Generator, shape, dist: str, mat: int, variant: int) -> np.ndarray:
    if variant == 1:
        return rng.integers(-8, 9, size=shape).astype(np.float64)
    if dist == "uniform":
        return 2.0 * rng.random(shape) - 1.0
    if dist == "scaled":
        return (2.0 * rng.random(shape) - 1.0) * (1e6 if mat == 0 else 1e-6)
    if dist == "normal":
        return rng.standard_normal(shape)
    if dist == "unit":  # paper protocol, U[0,1)
        return rng.random(shape)
    raise ValueError(dist)


def matrix(cfg: Config, mat: int, variant: int = 0, row0: int = 0, row1: Optional[int] = None,
           out: Optional[np.ndarray] = None) -> np.ndarray:
    """Rows [row0, row1) of A (mat=0, N x P) or B (mat=1, P x M) of config `cfg`."""
    rows, cols = (cfg.N, cfg.P) if mat == 0 else (cfg.P, cfg.M)
    row1 = rows if row1 is None else row1
    if not (0 <= row0 <= row1 <= rows):
        raise ValueError("bad row range")
    res = out if out is not None else np.empty((row1 - row0, cols), dtype=np.float64)
    c0, c1 = row0 // CHUNK, (row1 + CHUNK - 1) // CHUNK
    for c in range(c0, c1):
        lo, hi = c * CHUNK, min(rows, (c + 1) * CHUNK)
        blk = _draw(_chunk_rng(cfg.cfg_id, mat, variant, c), (hi - lo, cols), cfg.dist, mat, variant)
        a, b = max(lo, row0), min(hi, row1)
        res[a - row0:b - row0] = blk[a - lo:b - lo]
    return res


def operands(key: str, variant: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    cfg = CONFIGS[key]
    return matrix(cfg, 0, variant), matrix(cfg, 1, variant)


def custom(N: int, P: int, M: int, seed: int, dist: str = "uniform", variant: int = 0):
    """Small ad-hoc shapes for sweeps (ragged tails, odd P, ...)."""
    cfg = Config(f"x{seed}", 1000 + seed, N, P, M, dist, True)
    return matrix(cfg, 0, variant), matrix(cfg, 1, variant)


def paper_protocol(n: int, seed: int = 42) -> Tuple[np.ndarray, np.ndarray]:
    """C = A (8A), A an n x n random matrix (read as U[0,1), reading R13)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED, 0, seed])))
    A = rng.random((n, n))
    return A, 8.0 * A


def sample_positions(cfg_id: int, N: int, M: int, count: int, shard: int = 0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED, cfg_id, 99, shard])))
    return np.stack([rng.integers(0, N, count), rng.integers(0, M, count)], axis=1)


def shard_rows(N: int, world: int, rank: int) -> Tuple[int, int]:
    """Row block of rank `rank` out of `world`: [r*ceil(N/g), min(N, (r+1)*ceil(N/g)))."""
    per = (N + world - 1) // world
    lo = min(N, rank * per)
    return lo, min(N, lo + per)
