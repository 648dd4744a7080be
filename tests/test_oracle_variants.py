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
