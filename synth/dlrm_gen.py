"""Seeded DLRM-style embedding workloads (inputs only; no pooling/placement arithmetic).

Recipe (all a reading of PAPER.md P:250 "we use the data generator
in DLRM", which states no distribution, plus BASELINE.json's configs):

* Substreams.  Every (config, world size W, batch k, global table g) gets its own PCG64 stream
  seeded by a splitmix64 chain.  Only raw 64-bit words (``random_raw``) are drawn and converted
  here, so the data does not depend on NumPy's distribution code.
* Pooling factor L of bag (g, j): fixed P, or 1 + (x mod (2*Pbar - 1)) ~ Uniform{1..2Pbar-1}.
* Row indices: truncated Zipf(alpha) over ranks 1..R by inverse CDF (u = (x >> 11) * 2^-53),
  rank mapped to a row by a per-table bijection row = (A_g * (rank-1) + C_g) mod R, gcd(A_g,R)=1,
  so hot rows differ per table and are scattered.  alpha = 0 gives uniform indices.
  Duplicates inside a bag are allowed (each occurrence counts, R#6).
* Table values (procedural, counter-based): x = splitmix64(key ^ splitmix64(seed)),
  key = (g*2^23 + row)*2^10 + d;  fp32 mode: ((x >> 40) - 2^23) * 2^-23 in [-1, 1)
  (exact binary32 values);  exact-int mode: (x >> 60) - 8 in [-8, 7].
  The device fill kernel (synth/fill.cu) and the oracle (oracle/oracle.c) each implement this
  same generator independently; tests pin the three against each other.
"""
from __future__ import annotations

import dataclasses
import functools
import math
import zlib
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

BASE_SEED = 230506942          # the arXiv id, R#20
TABLE_SEED_SALT = 0x7AB1E5EED
_M64 = (1 << 64) - 1


def _splitmix64_int(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 over a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


@dataclasses.dataclass(frozen=True)
class ProblemConfig:
    """One synthetic workload at one world size W.

    T: tables per rank (tuple of W ints).  R: rows per table.  D: embedding dim.  B: global batch.
    pool: ("fixed", P) or ("uniform", Pbar) -> L ~ U{1..2Pbar-1}.  alpha: Zipf exponent.
    value_mode: 0 = fp32 grid values, 1 = exact small integers.  partition: W+1 prefix or None.
    """
    name: str
    W: int
    T: Tuple[int, ...]
    R: int
    D: int
    B: int
    pool: Tuple[str, int]
    alpha: float = 1.05
    value_mode: int = 0
    partition: Optional[Tuple[int, ...]] = None

    @property
    def G(self) -> int:
        return int(sum(self.T))

    @property
    def part(self) -> np.ndarray:
        if self.partition is not None:
            return np.asarray(self.partition, dtype=np.int64)
        return even_partition(self.B, self.W)

    def toff(self, r: int) -> int:
        return int(sum(self.T[:r]))

    @property
    def cfg_id(self) -> int:
        return zlib.crc32(self.name.encode())

    @property
    def table_seed(self) -> int:
        return _splitmix64_int(BASE_SEED ^ (self.cfg_id << 20) ^ TABLE_SEED_SALT ^ self.value_mode)

    def mean_pool(self) -> float:
        kind, p = self.pool
        return float(p)

    def expected_nnz_per_rank(self, r: int = 0) -> float:
        return self.T[r] * self.B * self.mean_pool()


def even_partition(B: int, W: int) -> np.ndarray:
    if B % W != 0:
        raise ValueError(f"even split needs B % W == 0 (B={B}, W={W}); pass a partition")
    return np.arange(W + 1, dtype=np.int64) * (B // W)


# BASELINE.json configs (DESIGN.md "Input recipe" gives the readings of unstated values).
CONFIGS: Dict[str, dict] = {
    "tiny": dict(W=2, T=4, R=1000, D=16, B=64, pool=("fixed", 4)),
    "dlrm_small": dict(W=8, T=8, R=1_000_000, D=64, B=2048, pool=("uniform", 20)),
    "dlrm_wide": dict(W=8, T=16, R=4_000_000, D=256, B=4096, pool=("uniform", 32)),
    **{f"sweep_p{p}": dict(W=8, T=16, R=2_000_000, D=128, B=8192, pool=("fixed", p))
       for p in (1, 2, 4, 8, 16, 32, 64, 128)},
    # weak scaling: per-GPU batch fixed at 1024 -> B = 1024 * W (B scales with W)
    "weak": dict(W=8, T=16, R=2_000_000, D=128, B=1024, pool=("uniform", 20), weak=True),
}


def config_for(name: str, W: Optional[int] = None, alpha: float = 1.05, value_mode: int = 0,
               **overrides) -> ProblemConfig:
    """Config `name` at world size W (W-scaling rule: keep T_r, R, D, B, Pbar; vary W;
    for 'weak' the per-GPU batch is fixed, so B = 1024 * W)."""
    base = dict(CONFIGS[name])
    weak = base.pop("weak", False)
    W = base["W"] if W is None else int(W)
    B = base["B"] * W if weak else base["B"]
    T = base["T"]
    kw = dict(name=name, W=W, T=tuple([T] * W), R=base["R"], D=base["D"], B=B,
              pool=base["pool"], alpha=alpha, value_mode=value_mode)
    kw.update(overrides)
    if isinstance(kw["T"], int):
        kw["T"] = tuple([kw["T"]] * kw["W"])
    return ProblemConfig(**kw)


@functools.lru_cache(maxsize=8)
def zipf_cdf(R: int, alpha: float) -> np.ndarray:
    """Cumulative (unnormalised) Zipf weights sum_{k<=n} k^-alpha, n = 1..R, float64."""
    k = np.arange(1, R + 1, dtype=np.float64)
    return np.cumsum(k ** (-alpha))


def _substream_seed(cfg: ProblemConfig, batch: int, g: int) -> int:
    h = _splitmix64_int(BASE_SEED ^ cfg.cfg_id)
    for v in (cfg.W, batch, g, int(round(cfg.alpha * 1000))):
        h = _splitmix64_int(h ^ v)
    return h


def _raw(bitgen: np.random.PCG64, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    return np.asarray(bitgen.random_raw(n), dtype=np.uint64)


def _bijection(R: int, a_raw: int, c_raw: int) -> Tuple[int, int]:
    A = (a_raw % R) | 1
    while math.gcd(A, R) != 1:
        A += 2
    return A % R if R > 1 else 0, c_raw % R


def gen_table_bags(cfg: ProblemConfig, batch: int, g: int) -> Tuple[np.ndarray, np.ndarray]:
    """Bags of global table g for all B samples: (lengths int64[B], rows int32[sum L])."""
    bg = np.random.PCG64(_substream_seed(cfg, batch, g))
    ac = _raw(bg, 2)
    A, C = _bijection(cfg.R, int(ac[0]), int(ac[1]))
    kind, p = cfg.pool
    if kind == "fixed":
        L = np.full(cfg.B, int(p), dtype=np.int64)
    elif kind == "uniform":
        L = (1 + (_raw(bg, cfg.B) % np.uint64(2 * p - 1))).astype(np.int64)
    elif kind == "list":   # explicit lengths (tests)
        raise ValueError("use gen_csr_from_lengths for explicit lengths")
    else:
        raise ValueError(kind)
    n = int(L.sum())
    x = _raw(bg, n)
    if cfg.alpha == 0.0:
        u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        rank0 = np.minimum((u * cfg.R).astype(np.int64), cfg.R - 1)
    else:
        cdf = zipf_cdf(cfg.R, cfg.alpha)
        u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        rank0 = np.searchsorted(cdf, u * cdf[-1], side="right").astype(np.int64)
        np.minimum(rank0, cfg.R - 1, out=rank0)
    rows = ((np.uint64(A) * rank0.astype(np.uint64) + np.uint64(C)) % np.uint64(cfg.R)).astype(np.int32)
    return L, rows


def gen_rank_csr(cfg: ProblemConfig, r: int, batch: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """Rank r's CSR: indices int32[nnz_r] (tables concatenated table-major) and
    offsets int32[T_r*B + 1] (absolute, offsets[0] = 0), R#8."""
    toff = cfg.toff(r)
    Ls, rows = [], []
    for t in range(cfg.T[r]):
        L, rw = gen_table_bags(cfg, batch, toff + t)
        Ls.append(L)
        rows.append(rw)
    if Ls:
        L = np.concatenate(Ls)
        idx = np.concatenate(rows).astype(np.int32)
    else:
        L = np.zeros(0, dtype=np.int64)
        idx = np.zeros(0, dtype=np.int32)
    if idx.size >= 2 ** 31:
        raise ValueError("nnz per rank must be < 2^31 (int32 offsets, R#8)")
    off = np.zeros(L.size + 1, dtype=np.int64)
    np.cumsum(L, out=off[1:])
    return idx, off.astype(np.int32)


def gen_all_csr(cfg: ProblemConfig, batch: int = 0) -> List[Tuple[np.ndarray, np.ndarray]]:
    return [gen_rank_csr(cfg, r, batch) for r in range(cfg.W)]


def table_values_host(seed: int, mode: int, g: int, R: int, D: int) -> np.ndarray:
    """Host copy of procedural table g, float32 [R, D] (small tables only)."""
    if R >= (1 << 23) or D > 1024:
        raise ValueError("procedural key needs R < 2^23 and D <= 1024")
    row = np.arange(R, dtype=np.uint64)[:, None]
    d = np.arange(D, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        key = (np.uint64(g) * np.uint64(1 << 23) + row) * np.uint64(1024) + d
    x = splitmix64_np(key ^ np.uint64(_splitmix64_int(seed)))
    if mode == 1:
        return ((x >> np.uint64(60)).astype(np.int64) - 8).astype(np.float32)
    if mode == 2:    # k * 2^-7, k in [-128, 127]: exact in bfloat16 and binary16
        return (((x >> np.uint64(56)).astype(np.int64) - 128).astype(np.float64) / 128.0).astype(np.float32)
    q = (x >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (q.astype(np.float64) * (2.0 ** -23)).astype(np.float32)


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 values that are exactly representable in bfloat16 -> uint16 bits (raises if not)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    if np.any(u & np.uint32(0xFFFF)):
        raise ValueError("values are not exactly representable in bfloat16")
    return (u >> np.uint32(16)).astype(np.uint16)


def to_f16_bits(a: np.ndarray) -> np.ndarray:
    """float32 values exactly representable in binary16 -> uint16 bits (raises if not)."""
    h = np.ascontiguousarray(a, dtype=np.float32).astype(np.float16)
    if not np.array_equal(h.astype(np.float32), a):
        raise ValueError("values are not exactly representable in binary16")
    return h.view(np.uint16)


def gen_weights(cfg: ProblemConfig, r: int, nnz: int, batch: int = 0, mode: int = 0) -> np.ndarray:
    """Per-sample weights for rank r's indices: mode 0 fp32 (x >> 40) * 2^-24 in [0, 1);
    mode 1 small integers in [-4, 3] (products and sums stay exact)."""
    bg = np.random.PCG64(_splitmix64_int(_substream_seed(cfg, batch, 1 << 30) ^ r))
    x = _raw(bg, nnz)
    if mode == 1:
        return ((x >> np.uint64(61)).astype(np.int64) - 4).astype(np.float32)
    return ((x >> np.uint64(40)).astype(np.float64) * 2.0 ** -24).astype(np.float32)
