"""Seeded inputs for the fused AllGather + GEMM.

Inputs only -- no gathering, no products, no sums.  Every element of every operand is a pure
function of (seed, tensor id, row, column), so either side can materialise any row it needs:

    x   = splitmix64(key ^ splitmix64(seed)),   key = ((tensor << 24) + row) << 16 | col
    mode 0 ("grid"):      ((x >> 57) - 64) * 2^-6       in [-1, 1), 7 significant bits
    mode 1 ("exact-int"): (x >> 61) - 4                  in [-4, 3]

Both modes are exactly representable in bfloat16 (8 significant bits), so the bf16 operand
holds exactly the value drawn here.  Tensor ids: X of rank r = 1000 + r, weight shard W_s of
rank s = 2000 + s (R#35).  row < 2^24, col < 2^16.

The device fill (synth/fill.cu ``synth_fill_gemm_bf16``) implements the same generator
independently; a GPU test pins the two against each other.
"""
from __future__ import annotations

import dataclasses
from typing import Tuple

import numpy as np

from .dlrm_gen import splitmix64_np

GEMM_SEED = 2305069420
X_TENSOR, W_TENSOR = 1000, 2000


def values(tensor: int, rows: np.ndarray, cols: np.ndarray, seed: int = GEMM_SEED,
           mode: int = 0) -> np.ndarray:
    """Element values (float64, each exactly a bf16 value) at the outer grid rows x cols."""
    rows = np.asarray(rows, dtype=np.uint64).reshape(-1, 1)
    cols = np.asarray(cols, dtype=np.uint64).reshape(1, -1)
    key = (((np.uint64(tensor) << np.uint64(24)) + rows) << np.uint64(16)) | cols
    s = splitmix64_np(np.asarray([seed], dtype=np.uint64))[0]
    x = splitmix64_np(key ^ s)
    if mode == 0:
        return ((x >> np.uint64(57)).astype(np.int64) - 64).astype(np.float64) * 2.0 ** -6
    if mode == 1:
        return ((x >> np.uint64(61)).astype(np.int64) - 4).astype(np.float64)
    raise ValueError(f"mode {mode}")


def matrix(tensor: int, nrows: int, ncols: int, seed: int = GEMM_SEED, mode: int = 0,
           row0: int = 0) -> np.ndarray:
    return values(tensor, np.arange(row0, row0 + nrows), np.arange(ncols), seed, mode)


@dataclasses.dataclass(frozen=True)
class GemmConfig:
    """One AllGather + GEMM workload at world size W (FSDP layer).

    Every rank r holds activations X_r [M][K] and the weight shard W_r [N_r][K] (rows
    r*N_r .. (r+1)*N_r of the layer's weight W [W*N_r][K]); it needs Y_r = X_r W^T [M][W*N_r].
    """
    name: str
    W: int
    M: int
    N_r: int
    K: int
    mode: int = 0

    @property
    def N(self) -> int:
        return self.W * self.N_r

    def flops_per_rank(self) -> float:
        return 2.0 * self.M * self.N * self.K


# Workloads (R#36): a tiny case the oracle finishes in seconds, and an FSDP
# transformer FFN up-projection (hidden 8192, FFN 28672, 8192 tokens per rank) with the weight
# sharded over the W ranks; the W-scaling rule keeps M, K and the FULL weight fixed.
GEMM_CONFIGS = {
    "ag_tiny": dict(M=256, N=1024, K=512),
    "ag_small": dict(M=2048, N=8192, K=4096),
    "ag_ffn": dict(M=8192, N=28672, K=8192),
}


def gemm_config(name: str, W: int, mode: int = 0) -> GemmConfig:
    c = GEMM_CONFIGS[name]
    if c["N"] % W:
        raise ValueError(f"{name}: N={c['N']} not divisible by W={W}")
    return GemmConfig(name, W, c["M"], c["N"] // W, c["K"], mode)


def rank_inputs(cfg: GemmConfig, r: int, seed: int = GEMM_SEED) -> Tuple[np.ndarray, np.ndarray]:
    """(X_r [M][K], W_r [N_r][K]) as float64 arrays of bf16-exact values."""
    return (matrix(X_TENSOR + r, cfg.M, cfg.K, seed, cfg.mode),
            matrix(W_TENSOR + r, cfg.N_r, cfg.K, seed, cfg.mode))


def to_bf16_bits_exact(a: np.ndarray) -> np.ndarray:
    """Bit patterns of values already exact in bf16 (asserted): the top half of the fp32 bits."""
    f = np.asarray(a, dtype=np.float32)
    if not np.array_equal(f.astype(np.float64), np.asarray(a, dtype=np.float64)):
        raise ValueError("value not exact in fp32")
    u = f.view(np.uint32)
    if np.any(u & np.uint32(0xFFFF)):
        raise ValueError("value not exact in bf16")
    return (u >> np.uint32(16)).astype(np.uint16)
