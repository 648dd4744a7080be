"""Problem builders shared by the CPU and GPU tests (inputs only, no method arithmetic)."""
from __future__ import annotations

import dataclasses
import json
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@dataclasses.dataclass
class Problem:
    W: int
    T: List[int]
    D: int
    B: int
    part: np.ndarray                   # W+1 prefix
    tables: List[np.ndarray]           # G arrays [rows_g, D] float32 (materialised)
    indices: List[np.ndarray]          # per rank int32
    offsets: List[np.ndarray]          # per rank int32 [T_r*B+1]
    cfg: Optional[synth.ProblemConfig] = None

    @property
    def G(self) -> int:
        return int(sum(self.T))

    def toff(self, r: int) -> int:
        return int(sum(self.T[:r]))

    def b(self, s: int) -> int:
        return int(self.part[s + 1] - self.part[s])

    def rank_tables(self, r: int) -> List[np.ndarray]:
        return self.tables[self.toff(r): self.toff(r) + self.T[r]]


def csr_from_bags(bags_per_table: Sequence[Sequence[Sequence[int]]]) -> Tuple[np.ndarray, np.ndarray]:
    """bags_per_table[t][j] = list of rows  ->  (indices int32, offsets int32[T*B+1])."""
    idx, off = [], [0]
    for bags in bags_per_table:
        for bag in bags:
            idx.extend(bag)
            off.append(len(idx))
    return np.asarray(idx, dtype=np.int32), np.asarray(off, dtype=np.int32)


def from_config(cfg: synth.ProblemConfig, batch: int = 0) -> Problem:
    csr = synth.gen_all_csr(cfg, batch)
    tables = [synth.table_values_host(cfg.table_seed, cfg.value_mode, g, cfg.R, cfg.D)
              for g in range(cfg.G)]
    return Problem(cfg.W, list(cfg.T), cfg.D, cfg.B, cfg.part, tables,
                   [c[0] for c in csr], [c[1] for c in csr], cfg)


def hand_example() -> Problem:
    gd = load_golden("hand_example.json")
    W, T, R, D, B = gd["W"], gd["T"], gd["R"], gd["D"], gd["B"]
    G = sum(T)
    tables = [np.array([[100 * g + 10 * row + d for d in range(D)] for row in range(R)],
                       dtype=np.float32) for g in range(G)]
    idx = [np.array(gd["csr"][f"rank{r}"]["indices"], np.int32) for r in range(W)]
    off = [np.array(gd["csr"][f"rank{r}"]["offsets"], np.int32) for r in range(W)]
    return Problem(W, list(T), D, B, synth.even_partition(B, W), tables, idx, off)


def random_partition(rng: np.random.Generator, B: int, W: int) -> np.ndarray:
    """Ragged contiguous blocks (some possibly empty) summing to B (R#1)."""
    cuts = np.sort(rng.integers(0, B + 1, size=W - 1))
    return np.concatenate([[0], cuts, [B]]).astype(np.int64)


def random_problem(seed: int, W: Optional[int] = None, value_mode: int = 0,
                   ragged: bool = False, max_B: int = 512, max_D: int = 256,
                   empty_bags: bool = True) -> Problem:
    """SPEC S:521-style random config: W in {1,2,4,8}, T_r in 1..8 (uneven across ranks),
    B in 8..max_B, D in 4..max_D step 4, mixed bag lengths including empty bags."""
    rng = np.random.default_rng(seed)
    W = int(rng.choice([1, 2, 4, 8])) if W is None else W
    T = [int(rng.integers(1, 9)) for _ in range(W)]
    D = int(rng.integers(1, max_D // 4 + 1)) * 4
    if ragged:
        B = int(rng.integers(8, max_B + 1))
        part = random_partition(rng, B, W)
    else:
        B = int(rng.integers(max(1, 8 // W), max_B // W + 1)) * W
        part = synth.even_partition(B, W)
    G = sum(T)
    R = [int(rng.integers(1, 300)) for _ in range(G)]
    if value_mode == 1:
        tables = [rng.integers(-8, 8, size=(R[g], D)).astype(np.float32) for g in range(G)]
    else:
        tables = [(rng.integers(-(1 << 23), 1 << 23, size=(R[g], D)) * 2.0 ** -23).astype(np.float32)
                  for g in range(G)]
    indices, offsets = [], []
    g = 0
    maxL = int(rng.choice([1, 4, 20, 64]))
    for r in range(W):
        bags_t = []
        for t in range(T[r]):
            lo = 0 if empty_bags else 1
            L = rng.integers(lo, maxL + 1, size=B)
            bags_t.append([list(rng.integers(0, R[g], size=l)) for l in L])
            g += 1
        i, o = csr_from_bags(bags_t)
        indices.append(i)
        offsets.append(o)
    return Problem(W, T, D, B, part, tables, indices, offsets)
