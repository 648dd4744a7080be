"""Pins for the oracle's f2 variants (mean pooling, per-sample weights, bf16/fp16 tables),
each against something other than the oracle itself."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth
from tests._problems import Problem, csr_from_bags, random_problem

U32 = 2.0 ** -24


def torch_concat(p: Problem, mode="sum", weights=None):
    cols = []
    for r in range(p.W):
        for t in range(p.T[r]):
            g = p.toff(r) + t
            off = p.offsets[r][t * p.B: (t + 1) * p.B + 1].astype(np.int64)
            idx = torch.from_numpy(p.indices[r][off[0]: off[-1]].astype(np.int64))
            psw = None
            if weights is not None:
                psw = torch.from_numpy(weights[r][off[0]: off[-1]])
            cols.append(F.embedding_bag(idx, torch.from_numpy(p.tables[g]),
                                        torch.from_numpy(off - off[0]), mode=mode,
                                        include_last_offset=True, per_sample_weights=psw).numpy())
    return np.concatenate(cols, axis=1)


def run(p, **kw):
    return np.concatenate(oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets,
                                         **kw), axis=0)


# ----------------------------------------------------------------------------- conversions

def test_bf16_conversion_all_bit_patterns():
    """bfloat16 is the top half of binary32: compare all 65536 patterns with numpy."""
    bits = np.arange(1 << 16, dtype=np.uint32)
    ref = (bits << np.uint32(16)).view(np.float32)
    got = np.array([oracle.bf16_to_float(int(b)) for b in bits], dtype=np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint32), ref[~nan].view(np.uint32))


def test_f16_conversion_all_bit_patterns():
    """IEEE binary16 -> binary32 (subnormals, +-0, inf, NaN) against numpy's float16."""
    bits = np.arange(1 << 16, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float32)
    got = np.array([oracle.f16_to_float(int(b)) for b in bits], dtype=np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint32), ref[~nan].view(np.uint32))


@pytest.mark.parametrize("dtype", [oracle.BF16, oracle.F16])
def test_half_tables_equal_fp32_tables_with_the_same_values(dtype):
    """Mode-2 values (k * 2^-7) are exact in bf16 and fp16, so the conversion is exact and the
    half-table result equals the fp32-table result bitwise."""
    cfg = synth.config_for("tiny", value_mode=2)
    tabs = [synth.table_values_host(cfg.table_seed, 2, g, cfg.R, cfg.D) for g in range(cfg.G)]
    conv = synth.to_bf16_bits if dtype == oracle.BF16 else synth.to_f16_bits
    csr = synth.gen_all_csr(cfg, 0)
    a = oracle.emb_a2a(cfg.part, cfg.D, cfg.B, cfg.T, tabs, [c[0] for c in csr], [c[1] for c in csr])
    b = oracle.emb_a2a(cfg.part, cfg.D, cfg.B, cfg.T, [conv(t) for t in tabs],
                       [c[0] for c in csr], [c[1] for c in csr], dtype=dtype)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_half_tables_vs_torch_on_general_values():
    """Arbitrary bf16/fp16 bit patterns (finite): oracle == torch embedding_bag over the
    up-converted float32 table, exact-int-free fp32 check within the summation bound."""
    rng = np.random.default_rng(3)
    p = random_problem(11, W=2, value_mode=0)
    for conv, dt in ((lambda a: (a.view(np.uint32) >> np.uint32(16)).astype(np.uint16), oracle.BF16),
                     (lambda a: a.astype(np.float16).view(np.uint16), oracle.F16)):
        half = [conv(t) for t in p.tables]
        up = [((h.astype(np.uint32) << np.uint32(16)).view(np.float32) if dt == oracle.BF16
               else h.view(np.float16).astype(np.float32)) for h in half]
        q = Problem(p.W, p.T, p.D, p.B, p.part, up, p.indices, p.offsets)
        got = np.concatenate(oracle.emb_a2a(p.part, p.D, p.B, p.T, half, p.indices, p.offsets,
                                            dtype=dt), axis=0)
        np.testing.assert_array_equal(got, run(q))
        np.testing.assert_allclose(got, torch_concat(q), rtol=1e-5, atol=1e-5)


# ----------------------------------------------------------------------------- mean pooling

@pytest.mark.parametrize("seed", range(4))
def test_mean_pooling_equals_torch_mean(seed):
    """P:119 (EmbeddingBag_..._sum_mean): torch's mean mode; empty bags give 0 in both."""
    p = random_problem(500 + seed, value_mode=0)
    np.testing.assert_allclose(run(p, pooling=oracle.MEAN), torch_concat(p, "mean"),
                               rtol=1e-6, atol=1e-7)


def test_mean_is_sum_divided_by_bag_length_exact_int():
    """Closed form in exact-int mode: mean = fl(sum / L), sums exact."""
    p = random_problem(41, value_mode=1)
    s = run(p)
    m = run(p, pooling=oracle.MEAN)
    L = np.zeros_like(s)
    for r in range(p.W):
        for t in range(p.T[r]):
            g = p.toff(r) + t
            o = p.offsets[r][t * p.B:(t + 1) * p.B + 1].astype(np.int64)
            L[:, g * p.D:(g + 1) * p.D] = np.diff(o)[:, None]
    want = np.where(L > 0, (s / np.maximum(L, 1)).astype(np.float32), 0).astype(np.float32)
    np.testing.assert_array_equal(m, want)
    assert not np.any(np.signbit(m[L == 0]))


# ----------------------------------------------------------------------------- weights

def _weights(p, mode):
    cfg = synth.config_for("tiny")
    return [synth.gen_weights(cfg, r, p.indices[r].size, mode=mode) for r in range(p.W)]


@pytest.mark.parametrize("seed", range(4))
def test_weighted_sum_equals_torch_exact_int(seed):
    """Integer tables and integer weights: products and sums are exact, so the oracle equals
    torch's per_sample_weights embedding_bag bitwise."""
    p = random_problem(600 + seed, value_mode=1)
    w = _weights(p, 1)
    np.testing.assert_array_equal(run(p, weights=w), torch_concat(p, "sum", w))


def test_weighted_sum_within_bound_fp32():
    p = random_problem(650, value_mode=0)
    w = _weights(p, 0)
    o32 = run(p, weights=w).astype(np.float64)
    o64 = run(p, weights=w, precision=64)
    ab = Problem(p.W, p.T, p.D, p.B, p.part, [np.abs(t) for t in p.tables], p.indices, p.offsets)
    mag = run(ab, weights=[np.abs(x) for x in w], precision=64)
    Lmax = max(int(np.diff(o).max()) if o.size > 1 else 0 for o in p.offsets)
    gam = 2 * Lmax * U32 / (1 - 2 * Lmax * U32)
    assert np.all(np.abs(o32 - o64) <= gam * mag)


def test_unit_weights_equal_unweighted_bitwise():
    p = random_problem(660, value_mode=0)
    w = [np.ones(i.size, np.float32) for i in p.indices]
    np.testing.assert_array_equal(run(p, weights=w), run(p))


def test_weights_with_mean_is_rejected():
    p = random_problem(661, value_mode=0)
    w = [np.ones(i.size, np.float32) for i in p.indices]
    with pytest.raises(oracle.OracleError):
        run(p, weights=w, pooling=oracle.MEAN)


def test_procedural_rows_ex_equal_materialised():
    cfg = synth.config_for("tiny", value_mode=2)
    csr = synth.gen_all_csr(cfg, 0)
    tabs = [synth.table_values_host(cfg.table_seed, 2, g, cfg.R, cfg.D) for g in range(cfg.G)]
    w = [synth.gen_weights(cfg, r, csr[r][0].size) for r in range(cfg.W)]
    for pooling, ww in ((oracle.MEAN, None), (oracle.SUM, w)):
        full = oracle.emb_a2a(cfg.part, cfg.D, cfg.B, cfg.T, tabs, [c[0] for c in csr],
                              [c[1] for c in csr], weights=ww, pooling=pooling)
        for s in range(cfg.W):
            b = int(cfg.part[s + 1] - cfg.part[s])
            rows = oracle.emb_a2a_rows(cfg.table_seed, 2, cfg.part, cfg.D, cfg.B, cfg.T, cfg.R,
                                       [c[0] for c in csr], [c[1] for c in csr], s, np.arange(b),
                                       weights=ww, pooling=pooling)
            np.testing.assert_array_equal(rows, full[s])


# ------------------------------------------------------------------ 16-bit output (R#32)

def _sweep_f32_patterns(seed=0):
    """Every 16-bit high half x low halves that sit on and around both types' rounding
    boundaries (bf16 ties at 0x8000, binary16 ties at bit 12 in the normal range and higher
    bits for subnormals), plus random patterns; NaN patterns dropped."""
    hi = np.arange(1 << 16, dtype=np.uint32) << np.uint32(16)
    lows = np.array([0x0000, 0x0001, 0x0FFF, 0x1000, 0x1001, 0x1FFF, 0x2000, 0x3000, 0x7FFF,
                     0x8000, 0x8001, 0xBFFF, 0xC000, 0xFFFF], dtype=np.uint32)
    pats = (hi[:, None] | lows[None, :]).ravel()
    rng = np.random.default_rng(seed)
    pats = np.concatenate([pats, rng.integers(0, 1 << 32, 400_000, dtype=np.uint64).astype(np.uint32)])
    f = pats.view(np.float32)
    return f[~np.isnan(f)]


def test_round_to_half_f16_equals_numpy():
    """Pin: numpy's float32 -> float16 cast rounds to nearest even (incl. subnormals, overflow
    to inf); the oracle's bisection over the binary16 patterns must agree on every pattern."""
    f = _sweep_f32_patterns(1)
    with np.errstate(over="ignore"):
        want = f.astype(np.float16).view(np.uint16)
    np.testing.assert_array_equal(oracle.round_to_half(f, oracle.F16), want)


def test_round_to_half_bf16_equals_torch():
    """Pin: torch's float32 -> bfloat16 conversion rounds to nearest even."""
    f = _sweep_f32_patterns(2)
    want = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(oracle.round_to_half(f, oracle.BF16), want)


@pytest.mark.parametrize("v,dt,bits", [
    (1.0 + 2.0 ** -8, oracle.BF16, 0x3F80),        # tie 1.0 | 1+2^-7 -> even (1.0)
    (1.0 + 3 * 2.0 ** -8, oracle.BF16, 0x3F82),    # tie 1+2^-7 | 1+2^-6 -> even
    (-(1.0 + 2.0 ** -9), oracle.BF16, 0xBF80),     # below half an ulp -> down, sign kept
    (65520.0, oracle.F16, 0x7C00),                 # tie 65504 (odd) | 2^16 -> inf (IEEE)
    (65519.0, oracle.F16, 0x7BFF),                 # below the tie: largest finite
    (2.0 ** -25, oracle.F16, 0x0000),              # tie 0 | smallest subnormal -> 0 (even)
    (3 * 2.0 ** -26, oracle.F16, 0x0001),          # 0.75 of the smallest subnormal -> up
    (-0.0, oracle.F16, 0x8000), (-0.0, oracle.BF16, 0x8000),
    (1.0 + 2.0 ** -11, oracle.F16, 0x3C00),        # tie 1.0 | 1+2^-10 -> even
    (2049.0, oracle.F16, 0x6800),                  # tie 2048 | 2050 -> 2048 (even)
])
def test_round_to_half_worked_cases(v, dt, bits):
    assert int(oracle.round_to_half(np.array([v], np.float32), dt)[0]) == bits


def test_half_output_is_the_rounded_fp32_result():
    """out_dtype = BF16 / F16: the fp32 definition rounded once.  On exact-int tables the sums
    are integers of magnitude < 2^11, exact in binary16 (and in bf16 below 2^8): the bits are
    then those of the exact integer sum (closed form, independent of the rounding code)."""
    rng = np.random.default_rng(77)
    W, T, B, D, R = 2, [2, 3], 8, 8, 11
    tables = [rng.integers(-8, 8, size=(R, D)).astype(np.float32) for _ in range(5)]
    idx, off = [], []
    for r in range(W):
        i, o = csr_from_bags([[list(rng.integers(0, R, size=rng.integers(0, 9))) for _ in range(B)]
                              for _ in range(T[r])])
        idx.append(i)
        off.append(o)
    part = synth.even_partition(B, W)
    f32 = oracle.emb_a2a(part, D, B, T, tables, idx, off)
    for dt in (oracle.F16, oracle.BF16):
        got = oracle.emb_a2a(part, D, B, T, tables, idx, off, out_dtype=dt)
        for s in range(W):
            assert got[s].dtype == np.uint16
            np.testing.assert_array_equal(got[s], oracle.round_to_half(f32[s], dt))
            if dt == oracle.F16:
                np.testing.assert_array_equal(got[s], f32[s].astype(np.float16).view(np.uint16))
            small = np.abs(f32[s]) < 256
            bf = torch.from_numpy(f32[s]).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
            if dt == oracle.BF16:
                np.testing.assert_array_equal(got[s][small], bf[small])
        rows = oracle.emb_a2a_rows(5, 1, part, D, B, T, R, idx, off, 1, np.arange(B // W),
                                   out_dtype=dt)
        full = oracle.emb_a2a_rows(5, 1, part, D, B, T, R, idx, off, 1, np.arange(B // W))
        np.testing.assert_array_equal(rows, oracle.round_to_half(full, dt))
